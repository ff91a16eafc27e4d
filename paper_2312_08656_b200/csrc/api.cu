// api.cu — the C-ABI of include/maxk.h: host-side validation, the work-plan builder and dispatch.
//
// The plan is the B200 redesign of the paper's O(n) warp-partition meta-data (§4.1,
// PAPER.md:493 §4.2): rows are cut into units of <= `chunk` edges; hub rows (degree >
// chunk) become chunk units whose partial rows are summed in chunk order by combine_kernel; all other
// rows are whole units.  Units are ordered longest-first so the kernels' dynamic warp scheduler
// approximates LPT (longest-processing-time-first) balance on power-law graphs.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include "maxk_internal.cuh"

namespace maxk {

namespace {
thread_local std::string g_detail;
std::atomic<uint64_t> g_launches{0};
}  // namespace

bool force_generic() {
  static const bool v = [] {
    const char* e = getenv("MAXK_FORCE_GENERIC");
    return e && e[0] == '1';
  }();
  return v;
}

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 1;
  }
  return cached[dev];
}

maxk_status_t fail(maxk_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_detail = buf;
  return s;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MAXK_PDL");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

maxk_status_t check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MAXK_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return MAXK_OK;
}

maxk_status_t resident_ctas(const void* kern, int threads, size_t smem, const char* name, int* per_sm) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  // occupancy per (kernel, threads, smem, device); the dynamic-smem limit is a property of the kernel alone,
  // so it is tracked per (kernel, device) and only ever raised (a smaller request must not lower it under a
  // cached larger one: ADVICE r01)
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> smem_limit;
  std::lock_guard<std::mutex> lock(mu);
  if (smem > 48 * 1024) {
    size_t& lim = smem_limit[std::make_pair(kern, dev)];
    if (smem > lim) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MAXK_ERR_CUDA, "%s: cudaFuncSetAttribute(%zu B): %s", name, smem, cudaGetErrorString(e));
      }
      lim = smem;
    }
  }
  const auto key = std::make_tuple(kern, threads, smem, dev);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *per_sm = it->second;
    return MAXK_OK;
  }
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem);
  if (e != cudaSuccess || n < 1) {
    cudaGetLastError();
    return fail(MAXK_ERR_CUDA, "%s: occupancy query failed (%s)", name, cudaGetErrorString(e));
  }
  cache[key] = n;
  *per_sm = n;
  return MAXK_OK;
}

namespace {

maxk_status_t check_widths(int32_t h, int32_t k, int32_t idx_bytes) {
  if (h < 1) return fail(MAXK_ERR_INVALID_ARGUMENT, "h=%d must be >= 1", h);
  if (k < 1 || k > h) return fail(MAXK_ERR_INVALID_ARGUMENT, "k=%d must satisfy 1 <= k <= h=%d", k, h);
  if (idx_bytes == 1) {
    if (h > 256) return fail(MAXK_ERR_INVALID_ARGUMENT, "idx_bytes=1 requires h <= 256 (h=%d)", h);
  } else if (idx_bytes == 2) {
    if (h > 65536) return fail(MAXK_ERR_INVALID_ARGUMENT, "idx_bytes=2 requires h <= 65536 (h=%d)", h);
  } else {
    return fail(MAXK_ERR_INVALID_ARGUMENT, "idx_bytes=%d must be 1 or 2", idx_bytes);
  }
  return MAXK_OK;
}

maxk_status_t check_agg(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                        int64_t n_cols, int64_t nnz, const void* sp_idx, int32_t h, int32_t k, int32_t idx_bytes,
                        const void* dense, int64_t ld, const maxk_plan_t* plan) {
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0 || n_cols < 0 || nnz < 0)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "negative size (n_rows=%lld n_cols=%lld nnz=%lld)", (long long)n_rows,
                (long long)n_cols, (long long)nnz);
  if (n_cols > INT32_MAX) return fail(MAXK_ERR_UNSUPPORTED, "n_cols=%lld > INT32_MAX", (long long)n_cols);
  if (n_rows > INT32_MAX) return fail(MAXK_ERR_UNSUPPORTED, "n_rows=%lld > INT32_MAX", (long long)n_rows);
  if (h > 4096) return fail(MAXK_ERR_UNSUPPORTED, "h=%d > 4096 (shared-memory row buffer limit)", h);
  if (k > 1024) return fail(MAXK_ERR_UNSUPPORTED, "k=%d > 1024 (register-tiled CBSR row limit of this build)", k);
  if (ld < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "leading dimension %lld < h=%d", (long long)ld, h);
  if (n_rows > 0 && (!row_ptr || !dense)) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL row_ptr or dense operand");
  if (nnz > 0 && (!col_idx || !val || !sp_idx))
    return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL col_idx, val or sp_idx with nnz > 0");
  if (nnz > 0 && n_cols == 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "nnz > 0 with n_cols == 0");
  if (plan) {
    if (plan->n_rows != n_rows || plan->nnz != nnz)
      return fail(MAXK_ERR_INVALID_ARGUMENT, "plan built for n_rows=%lld nnz=%lld, called with n_rows=%lld nnz=%lld",
                  (long long)plan->n_rows, (long long)plan->nnz, (long long)n_rows, (long long)nnz);
    if (plan->h < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "plan built for h=%d < h=%d", plan->h, h);
    int dev = 0;
    cudaGetDevice(&dev);
    if (plan->device != dev)
      return fail(MAXK_ERR_INVALID_ARGUMENT, "plan belongs to device %d, current device is %d", plan->device, dev);
  }
  return MAXK_OK;
}

// Warps resident on the whole device for the aggregation kernels (8-warp CTAs, up to 8 per SM).
int64_t device_warps() { return (int64_t)sm_count() * 64; }

}  // namespace
}  // namespace maxk

using namespace maxk;

extern "C" {

const char* maxk_status_string(maxk_status_t s) {
  switch (s) {
    case MAXK_OK: return "MAXK_OK";
    case MAXK_ERR_INVALID_ARGUMENT: return "MAXK_ERR_INVALID_ARGUMENT";
    case MAXK_ERR_UNSUPPORTED: return "MAXK_ERR_UNSUPPORTED";
    case MAXK_ERR_CUDA: return "MAXK_ERR_CUDA";
    case MAXK_ERR_OUT_OF_MEMORY: return "MAXK_ERR_OUT_OF_MEMORY";
  }
  return "MAXK_ERR_UNKNOWN";
}

const char* maxk_last_error_detail(void) { return g_detail.c_str(); }

uint64_t maxk_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* maxk_version(void) { return "maxk-b200 0.1 sm_100a"; }

maxk_status_t maxk_topk_cbsr(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k, int32_t idx_bytes,
                             float* sp_data, void* sp_idx, maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_x < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x=%lld < h=%d", (long long)ld_x, h);
  if (h > 1024) return fail(MAXK_ERR_UNSUPPORTED, "top-k supports h <= 1024 (h=%d)", h);
  if (n_rows == 0) return MAXK_OK;
  if (!x || !sp_data || !sp_idx) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  return launch_topk(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, (cudaStream_t)stream);
}

static maxk_status_t topk_pairs_entry(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                   int32_t idx_bytes, float* sp_data, void* sp_idx, void* sp_pairs,
                                   maxk_stream_t stream, bool balanced) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_x < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x=%lld < h=%d", (long long)ld_x, h);
  if (k != 8 && k != 16) return fail(MAXK_ERR_UNSUPPORTED, "pair layout: k=%d not in {8, 16}", k);
  if (balanced && k != 16) return fail(MAXK_ERR_UNSUPPORTED, "balanced pair layout: k=%d != 16", k);
  if (n_rows == 0) return MAXK_OK;
  if (!x || !sp_data || !sp_idx || !sp_pairs)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  if ((reinterpret_cast<uintptr_t>(sp_pairs) & 15u) != 0)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "sp_pairs must be 16-byte aligned");
  return launch_topk_pairs(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, static_cast<uint2*>(sp_pairs),
                           (cudaStream_t)stream, balanced);
}

maxk_status_t maxk_topk_cbsr_pairs(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                   int32_t idx_bytes, float* sp_data, void* sp_idx, void* sp_pairs,
                                   maxk_stream_t stream) {
  return topk_pairs_entry(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, sp_pairs, stream, false);
}

maxk_status_t maxk_topk_cbsr_pairs_banked(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                          int32_t idx_bytes, float* sp_data, void* sp_idx, void* sp_pairs,
                                          maxk_stream_t stream) {
  return topk_pairs_entry(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, sp_pairs, stream, true);
}

maxk_status_t maxk_topk_cbsr_banked(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                    int32_t idx_bytes, float* sp_data, void* sp_idx, float* sp_bdata,
                                    void* sp_bidx, maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_x < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x=%lld < h=%d", (long long)ld_x, h);
  if (k != 32 && k != 64 && k != 128) return fail(MAXK_ERR_UNSUPPORTED, "banked order: k=%d not in {32, 64, 128}", k);
  if (h != 128 && h != 256 && h != 384 && h != 512)
    return fail(MAXK_ERR_UNSUPPORTED, "banked order: h=%d not in {128, 256, 384, 512}", h);
  if (n_rows == 0) return MAXK_OK;
  if (!x || !sp_data || !sp_idx || !sp_bdata || !sp_bidx)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  return launch_topk_banked(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, sp_bdata, sp_bidx,
                            (cudaStream_t)stream);
}

int32_t maxk_spgemm_fwd_replicated(int64_t n_rows, int64_t nnz, int32_t h, int32_t k) {
  // k = 16: the pair-layout forward's decision (the layer path reads the pair layout there)
  return n_rows > 0 && fwd_policy(n_rows, nnz, h, k, k == 16) == 1 ? 1 : 0;
}

maxk_status_t maxk_topk_cbsr_multi(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                   int32_t idx_bytes, int32_t n_dst, float* const* sp_data, void* const* sp_idx,
                                   maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_x < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x=%lld < h=%d", (long long)ld_x, h);
  if (n_dst < 1 || n_dst > 8) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_dst=%d not in [1, 8]", n_dst);
  if (!sp_data || !sp_idx) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL destination array");
  if (k != 8 && k != 16 && k != 32 && k != 64)
    return fail(MAXK_ERR_UNSUPPORTED, "topk multi: k=%d not in {8, 16, 32, 64}", k);
  if (h != 128 && h != 256) return fail(MAXK_ERR_UNSUPPORTED, "topk multi: h=%d not in {128, 256}", h);
  if (n_rows == 0) return MAXK_OK;
  if (!x) return fail(MAXK_ERR_INVALID_ARGUMENT, "x is NULL with n_rows > 0");
  for (int i = 0; i < n_dst; ++i)
    if (!sp_data[i] || !sp_idx[i]) return fail(MAXK_ERR_INVALID_ARGUMENT, "destination %d is NULL", i);
  Replicas rep{};
  rep.n = n_dst - 1;
  for (int i = 1; i < n_dst; ++i) {
    rep.data[i - 1] = sp_data[i];
    rep.idx[i - 1] = sp_idx[i];
  }
  return launch_topk_multi(x, n_rows, h, ld_x, k, idx_bytes, sp_data[0], sp_idx[0], rep, (cudaStream_t)stream);
}

maxk_status_t maxk_topk_cbsr_probe_stats(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                         int32_t idx_bytes, float* sp_data, void* sp_idx, int32_t* probes,
                                         maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_x < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x=%lld < h=%d", (long long)ld_x, h);
  if (n_rows == 0) return MAXK_OK;
  if (!x || !sp_data || !sp_idx || !probes) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  return launch_topk_probe_stats(x, n_rows, h, ld_x, k, idx_bytes, sp_data, sp_idx, probes, (cudaStream_t)stream);
}

maxk_status_t maxk_cbsr_scatter(const float* d_sp_data, const void* sp_idx, int64_t n_rows, int32_t h, int32_t k,
                                int32_t idx_bytes, float* dx, int64_t ld_dx, maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n_rows=%lld < 0", (long long)n_rows);
  if (ld_dx < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_dx=%lld < h=%d", (long long)ld_dx, h);
  if (h > 4096) return fail(MAXK_ERR_UNSUPPORTED, "h=%d > 4096", h);
  if (n_rows == 0) return MAXK_OK;
  if (!d_sp_data || !sp_idx || !dx) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  return launch_cbsr_scatter(d_sp_data, sp_idx, n_rows, h, k, idx_bytes, dx, ld_dx, (cudaStream_t)stream);
}

maxk_status_t maxk_linear_topk_cbsr(const void* x, int64_t n_rows, int32_t f_in, int64_t ld_x, const void* w_t,
                                    int64_t ld_w, const float* bias, int32_t h, int32_t k, int32_t idx_bytes,
                                    float* sp_data, void* sp_idx, float* z_out, int64_t ld_z, maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_widths(h, k, idx_bytes);
  if (s != MAXK_OK) return s;
  if (n_rows < 0 || f_in < 1) return fail(MAXK_ERR_INVALID_ARGUMENT, "bad n_rows=%lld or f_in=%d", (long long)n_rows, f_in);
  if (h != 128 && h != 256) return fail(MAXK_ERR_UNSUPPORTED, "linear_topk supports h in {128, 256} (h=%d)", h);
  if (f_in % 64 != 0 || (int64_t)f_in * h * 2 > 131072)
    return fail(MAXK_ERR_UNSUPPORTED, "linear_topk needs f_in %% 64 == 0 and f_in*h*2 <= 128 KiB (f_in=%d, h=%d)",
                f_in, h);
  if (k > 64) return fail(MAXK_ERR_UNSUPPORTED, "linear_topk supports k <= 64 (k=%d)", k);
  if (ld_x < f_in || ld_w < f_in) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x / ld_w < f_in");
  if (ld_x % 8 != 0 || ld_w % 8 != 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_x and ld_w must be multiples of 8");
  if (z_out && ld_z < h) return fail(MAXK_ERR_INVALID_ARGUMENT, "ld_z=%lld < h=%d", (long long)ld_z, h);
  if (z_out && (((uintptr_t)z_out & 15u) != 0 || ld_z % 4 != 0))
    return fail(MAXK_ERR_INVALID_ARGUMENT, "z_out must be 16-byte aligned with ld_z a multiple of 4");
  if (n_rows == 0) return MAXK_OK;
  if (!x || !w_t || !sp_data || !sp_idx) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n_rows > 0");
  if ((reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(w_t) & 15u))
    return fail(MAXK_ERR_INVALID_ARGUMENT, "x and w_t must be 16-byte aligned");
  return launch_linear_topk(x, n_rows, f_in, ld_x, w_t, ld_w, bias, h, k, idx_bytes, sp_data, sp_idx, z_out, ld_z,
                            (cudaStream_t)stream);
}

maxk_status_t maxk_plan_create(const int64_t* row_ptr, int64_t n_rows, int64_t nnz, int32_t h, int32_t k,
                               maxk_stream_t stream, maxk_plan_t** out) {
  g_detail.clear();
  if (!out) return fail(MAXK_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n_rows < 0 || nnz < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "negative n_rows or nnz");
  if (n_rows > INT32_MAX) return fail(MAXK_ERR_UNSUPPORTED, "n_rows > INT32_MAX");
  if (h < 1 || k < 1 || k > h) return fail(MAXK_ERR_INVALID_ARGUMENT, "bad h=%d k=%d", h, k);
  if (!row_ptr) return fail(MAXK_ERR_INVALID_ARGUMENT, "row_ptr is NULL");
  cudaStream_t st = (cudaStream_t)stream;

  std::vector<int64_t> rp((size_t)n_rows + 1);
  cudaError_t e = cudaMemcpyAsync(rp.data(), row_ptr, rp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(MAXK_ERR_CUDA, "plan: row_ptr copy: %s", cudaGetErrorString(e));
  for (int64_t i = 0; i < n_rows; ++i)
    if (rp[i + 1] < rp[i]) return fail(MAXK_ERR_INVALID_ARGUMENT, "row_ptr not monotone at row %lld", (long long)i);
  if (rp[n_rows] - rp[0] != nnz)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "nnz=%lld != row_ptr[n]-row_ptr[0]=%lld", (long long)nnz,
                (long long)(rp[n_rows] - rp[0]));

  // chunk: ~1/4 of the mean per-warp share, clamped to [256, 2048] edges, a multiple of 32
  int64_t chunk = nnz / (4 * device_warps());
  chunk = std::max<int64_t>(256, std::min<int64_t>(2048, chunk));
  chunk = (chunk + 31) / 32 * 32;

  std::vector<int32_t> hubs;
  int64_t max_deg = 0;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t d = rp[i + 1] - rp[i];
    max_deg = std::max(max_deg, d);
    if (d > chunk) hubs.push_back((int32_t)i);
  }
  std::stable_sort(hubs.begin(), hubs.end(),
                   [&](int32_t a, int32_t b) { return rp[a + 1] - rp[a] > rp[b + 1] - rp[b]; });
  std::vector<Unit> units;
  std::vector<Combine> comb;
  units.reserve((size_t)n_rows + (size_t)(nnz / chunk) + 1);
  for (int32_t r : hubs) {
    Combine cb;
    cb.u0 = (int64_t)units.size();
    cb.row = r;
    cb.n_chunks = 0;
    for (int64_t e0 = rp[r]; e0 < rp[r + 1]; e0 += chunk) {
      Unit u;
      u.e0 = e0;
      u.row = r;
      u.len = (int32_t)std::min<int64_t>(chunk, rp[r + 1] - e0);
      units.push_back(u);
      cb.n_chunks++;
    }
    comb.push_back(cb);
  }
  const int64_t n_chunk_units = (int64_t)units.size();
  // whole rows, degree-descending, ties by row id (counting sort over degree <= chunk)
  std::vector<int64_t> cnt((size_t)chunk + 2, 0);
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t d = rp[i + 1] - rp[i];
    if (d <= chunk) cnt[(size_t)(chunk - d)]++;
  }
  std::vector<int64_t> start((size_t)chunk + 2, 0);
  for (size_t b = 1; b < start.size(); ++b) start[b] = start[b - 1] + cnt[b - 1];
  const size_t n_whole = (size_t)start.back();
  std::vector<Unit> whole(n_whole);
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t d = rp[i + 1] - rp[i];
    if (d > chunk) continue;
    Unit u;
    u.e0 = rp[i];
    u.row = (int32_t)i;
    u.len = (int32_t)d;
    whole[(size_t)start[(size_t)(chunk - d)]++] = u;
  }
  units.insert(units.end(), whole.begin(), whole.end());

  maxk_plan* p = new maxk_plan();
  p->n_rows = n_rows;
  p->nnz = nnz;
  p->row_base = rp[0];
  p->h = h;
  p->k = k;
  p->chunk = chunk;
  p->n_units = (int64_t)units.size();
  p->n_chunk_units = n_chunk_units;
  p->n_split_rows = (int64_t)comb.size();
  {  // whole-row units are degree-descending: the short tail starts at the first unit with <= kShortLen edges
    int64_t us = (int64_t)units.size();
    for (int64_t u = n_chunk_units; u < (int64_t)units.size(); ++u)
      if (units[(size_t)u].len <= kShortLen) { us = u; break; }
    p->u_short = us;
  }
  cudaGetDevice(&p->device);
  auto oom = [&](const char* what, cudaError_t err) {
    maxk_plan_destroy(p);
    return fail(err == cudaErrorMemoryAllocation ? MAXK_ERR_OUT_OF_MEMORY : MAXK_ERR_CUDA, "plan: %s: %s", what,
                cudaGetErrorString(err));
  };
  if (!units.empty()) {
    e = cudaMalloc(&p->d_units, units.size() * sizeof(Unit));
    if (e != cudaSuccess) return oom("units", e);
    e = cudaMemcpyAsync(p->d_units, units.data(), units.size() * sizeof(Unit), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return oom("units copy", e);
  }
  if (!comb.empty()) {
    e = cudaMalloc(&p->d_combine, comb.size() * sizeof(Combine));
    if (e != cudaSuccess) return oom("combine", e);
    e = cudaMemcpyAsync(p->d_combine, comb.data(), comb.size() * sizeof(Combine), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return oom("combine copy", e);
    e = cudaMalloc(&p->d_partial, (size_t)n_chunk_units * (size_t)h * sizeof(float));
    if (e != cudaSuccess) return oom("partial", e);
  }
  e = cudaMalloc(&p->d_sched, 2 * kSchedWords * sizeof(unsigned));
  if (e != cudaSuccess) return oom("sched", e);
  e = cudaMemsetAsync(p->d_sched, 0, 2 * kSchedWords * sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return oom("upload", e);
  *out = p;
  return MAXK_OK;
}

void maxk_plan_destroy(maxk_plan_t* p) {
  if (!p) return;
  if (p->d_units) cudaFree(p->d_units);
  if (p->d_combine) cudaFree(p->d_combine);
  if (p->d_partial) cudaFree(p->d_partial);
  if (p->d_sched) cudaFree(p->d_sched);
  delete p;
}

maxk_status_t maxk_plan_info(const maxk_plan_t* p, int64_t* n_units, int64_t* n_split_rows, int64_t* chunk_edges,
                             int64_t* n_chunk_units) {
  g_detail.clear();
  if (!p) return fail(MAXK_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (n_units) *n_units = p->n_units;
  if (n_split_rows) *n_split_rows = p->n_split_rows;
  if (chunk_edges) *chunk_edges = p->chunk;
  if (n_chunk_units) *n_chunk_units = p->n_chunk_units;
  return MAXK_OK;
}

}  // extern "C"

namespace {

maxk_status_t spgemm_fwd_impl(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                              int64_t n_cols, int64_t nnz, const float* sp_data, const void* sp_idx, int32_t h,
                              int32_t k, int32_t idx_bytes, float* y, int64_t ld_y, const maxk_plan_t* plan,
                              maxk_stream_t stream, int accumulate, const void* pairs = nullptr) {
  g_detail.clear();
  maxk_status_t s =
      check_agg(row_ptr, col_idx, val, n_rows, n_cols, nnz, pairs ? pairs : sp_idx, h, k, idx_bytes, y, ld_y, plan);
  if (s != MAXK_OK) return s;
  if (nnz > 0 && !sp_data && !pairs) return fail(MAXK_ERR_INVALID_ARGUMENT, "sp_data is NULL with nnz > 0");
  if (n_rows == 0) return MAXK_OK;
  AggArgs a{};
  a.row_ptr = row_ptr;
  a.col = col_idx;
  a.val = val;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.nnz = nnz;
  a.sp_data = sp_data;
  a.sp_idx = sp_idx;
  a.h = h;
  a.k = k;
  a.y = y;
  a.ld_y = ld_y;
  a.accumulate = accumulate;
  a.pairs = static_cast<const uint2*>(pairs);
  if (plan) {
    a.units = plan->d_units;
    a.n_units = plan->n_units;
    a.n_chunk_units = plan->n_chunk_units;
    a.u_short = plan->u_short;
    a.partial = plan->d_partial;
    a.sched = plan->d_sched;
  } else {
    a.units = nullptr;
    a.n_units = n_rows;
    a.u_short = n_rows;
    a.n_chunk_units = 0;
    a.partial = nullptr;
    a.sched = nullptr;
  }
  return launch_spgemm_fwd(a, idx_bytes, plan, (cudaStream_t)stream);
}

maxk_status_t sspmm_bwd_impl(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                             int64_t n_cols, int64_t nnz, const float* dy, int64_t ld_dy, const void* sp_idx,
                             int32_t h, int32_t k, int32_t idx_bytes, float* d_sp_data, const maxk_plan_t* plan,
                             maxk_stream_t stream, int accumulate) {
  g_detail.clear();
  maxk_status_t s = check_agg(row_ptr, col_idx, val, n_rows, n_cols, nnz, sp_idx, h, k, idx_bytes, dy, ld_dy, plan);
  if (s != MAXK_OK) return s;
  if (n_cols > 0 && !d_sp_data) return fail(MAXK_ERR_INVALID_ARGUMENT, "d_sp_data is NULL with n_cols > 0");
  AggArgs a{};
  a.row_ptr = row_ptr;
  a.col = col_idx;
  a.val = val;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.nnz = nnz;
  a.sp_idx = sp_idx;
  a.h = h;
  a.k = k;
  a.dy = dy;
  a.ld_dy = ld_dy;
  a.d_sp_data = d_sp_data;
  a.accumulate = accumulate;
  if (plan) {
    a.units = plan->d_units;
    a.n_units = plan->n_units;
    a.n_chunk_units = plan->n_chunk_units;
    a.u_short = plan->u_short;
    a.sched = plan->d_sched + kSchedWords;
  } else {
    a.units = nullptr;
    a.n_units = nnz > 0 ? n_rows : 0;
    a.u_short = a.n_units;
    a.sched = nullptr;
  }
  if (nnz == 0) a.n_units = a.u_short = 0;
  return launch_sspmm_bwd(a, idx_bytes, (cudaStream_t)stream);
}

}  // namespace

extern "C" {

maxk_status_t maxk_spgemm_fwd(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                              int64_t n_cols, int64_t nnz, const float* sp_data, const void* sp_idx, int32_t h,
                              int32_t k, int32_t idx_bytes, float* y, int64_t ld_y, const maxk_plan_t* plan,
                              maxk_stream_t stream) {
  return spgemm_fwd_impl(row_ptr, col_idx, val, n_rows, n_cols, nnz, sp_data, sp_idx, h, k, idx_bytes, y, ld_y, plan,
                         stream, 0);
}

maxk_status_t maxk_spgemm_fwd_acc(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                                  int64_t n_cols, int64_t nnz, const float* sp_data, const void* sp_idx, int32_t h,
                                  int32_t k, int32_t idx_bytes, float* y, int64_t ld_y, const maxk_plan_t* plan,
                                  maxk_stream_t stream) {
  return spgemm_fwd_impl(row_ptr, col_idx, val, n_rows, n_cols, nnz, sp_data, sp_idx, h, k, idx_bytes, y, ld_y, plan,
                         stream, 1);
}

maxk_status_t maxk_spgemm_fwd_pairs(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                    int64_t n_rows, int64_t n_cols, int64_t nnz, const void* sp_pairs, int32_t h,
                                    int32_t k, float* y, int64_t ld_y, const maxk_plan_t* plan,
                                    maxk_stream_t stream) {
  g_detail.clear();
  if (k != 8 && k != 16) return fail(MAXK_ERR_UNSUPPORTED, "pair layout: k=%d not in {8, 16}", k);
  if (h > 65536) return fail(MAXK_ERR_INVALID_ARGUMENT, "h=%d > 65536", h);
  if (nnz > 0 && (reinterpret_cast<uintptr_t>(sp_pairs) & 15u) != 0)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "sp_pairs must be 16-byte aligned");
  return spgemm_fwd_impl(row_ptr, col_idx, val, n_rows, n_cols, nnz, nullptr, nullptr, h, k, h <= 256 ? 1 : 2, y,
                         ld_y, plan, stream, 0, sp_pairs);
}

maxk_status_t maxk_sspmm_bwd(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                             int64_t n_cols, int64_t nnz, const float* dy, int64_t ld_dy, const void* sp_idx,
                             int32_t h, int32_t k, int32_t idx_bytes, float* d_sp_data, const maxk_plan_t* plan,
                             maxk_stream_t stream) {
  return sspmm_bwd_impl(row_ptr, col_idx, val, n_rows, n_cols, nnz, dy, ld_dy, sp_idx, h, k, idx_bytes, d_sp_data,
                        plan, stream, 0);
}

maxk_status_t maxk_sspmm_bwd_acc(const int64_t* row_ptr, const int32_t* col_idx, const float* val, int64_t n_rows,
                                 int64_t n_cols, int64_t nnz, const float* dy, int64_t ld_dy, const void* sp_idx,
                                 int32_t h, int32_t k, int32_t idx_bytes, float* d_sp_data, const maxk_plan_t* plan,
                                 maxk_stream_t stream) {
  return sspmm_bwd_impl(row_ptr, col_idx, val, n_rows, n_cols, nnz, dy, ld_dy, sp_idx, h, k, idx_bytes, d_sp_data,
                        plan, stream, 1);
}

maxk_status_t maxk_sspmm_bwd_owners(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                    int64_t n_rows, int64_t n_cols, int64_t nnz, const float* dy, int64_t ld_dy,
                                    const void* sp_idx, int32_t h, int32_t k, int32_t idx_bytes, int32_t n_owners,
                                    int64_t owner_rows, float* const* d_owner, const maxk_plan_t* plan,
                                    maxk_stream_t stream) {
  g_detail.clear();
  maxk_status_t s = check_agg(row_ptr, col_idx, val, n_rows, n_cols, nnz, sp_idx, h, k, idx_bytes, dy, ld_dy, plan);
  if (s != MAXK_OK) return s;
  if (n_owners < 1 || owner_rows < 1 || n_cols != (int64_t)n_owners * owner_rows)
    return fail(MAXK_ERR_INVALID_ARGUMENT, "owners: n_cols=%lld != n_owners=%d x owner_rows=%lld", (long long)n_cols,
                n_owners, (long long)owner_rows);
  if (owner_rows >= (1ll << 24))
    return fail(MAXK_ERR_UNSUPPORTED, "owners: owner_rows=%lld >= 2^24", (long long)owner_rows);
  if (!d_owner) return fail(MAXK_ERR_INVALID_ARGUMENT, "d_owner is NULL");
  AggArgs a{};
  a.row_ptr = row_ptr;
  a.col = col_idx;
  a.val = val;
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.nnz = nnz;
  a.sp_idx = sp_idx;
  a.h = h;
  a.k = k;
  a.dy = dy;
  a.ld_dy = ld_dy;
  a.d_sp_data = nullptr;
  a.accumulate = 1;  // the owners' blocks are zeroed (or accumulated into) by their owners
  a.owner_dst = d_owner;
  a.owner_rows = owner_rows;
  a.n_owners = n_owners;
  a.owner_inv = 1.0f / (float)owner_rows;
  if (force_generic() || !vec_path_ok(a, false))
    return fail(MAXK_ERR_UNSUPPORTED, "owners: k=%d / alignment has no vector backward", k);
  if (plan) {
    a.units = plan->d_units;
    a.n_units = plan->n_units;
    a.n_chunk_units = plan->n_chunk_units;
    a.u_short = plan->u_short;
    a.sched = plan->d_sched + kSchedWords;
  } else {
    a.units = nullptr;
    a.n_units = nnz > 0 ? n_rows : 0;
    a.u_short = a.n_units;
    a.sched = nullptr;
  }
  if (nnz == 0) return MAXK_OK;
  return launch_sspmm_bwd(a, idx_bytes, (cudaStream_t)stream);
}

maxk_status_t maxk_add_f32(float* dst, const float* src, int64_t n, maxk_stream_t stream) {
  g_detail.clear();
  if (n < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "n=%lld < 0", (long long)n);
  if (n == 0) return MAXK_OK;
  if (!dst || !src) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  return launch_add(dst, src, n, (cudaStream_t)stream);
}

}  // extern "C"
