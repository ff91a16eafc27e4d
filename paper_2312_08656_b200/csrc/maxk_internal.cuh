// maxk_internal.cuh — device helpers and internal launcher declarations shared by the csrc/ kernels.
// Product code only: nothing here is shared with oracle/ (DESIGN.md §4).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "maxk.h"

namespace maxk {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------------------------
// Work plan.  A unit is a run of <= chunk edges of one CSR row.
//   units[0, n_chunk_units)        chunks of hub rows (deg > chunk), each row's chunks contiguous;
//                                  the forward writes their partial rows to partial[u * h].
//   units[n_chunk_units, n_units)  whole rows (deg <= chunk, including empty rows), degree-descending;
//                                  the forward writes y[row] directly.
// combine[s] lists, for hub row s, its chunk units [u0, u0 + n_chunks) summed in order into y[row].
// ---------------------------------------------------------------------------------------------
struct Unit {
  int64_t e0;   // first edge (absolute index into col_idx / val)
  int32_t row;  // local row id
  int32_t len;  // number of edges
};
static_assert(sizeof(Unit) == 16, "Unit is 16 bytes");

struct Combine {
  int64_t u0;        // first chunk unit
  int32_t row;       // local row id
  int32_t n_chunks;  // number of chunk units
};

}  // namespace maxk

struct maxk_plan {
  int64_t n_rows = 0, nnz = 0, row_base = 0;
  int32_t h = 0, k = 0;
  int64_t chunk = 0;
  int64_t n_units = 0, n_chunk_units = 0, n_split_rows = 0;
  int64_t u_short = 0;             // first unit with <= maxk::kShortLen edges (units are degree-sorted)
  maxk::Unit* d_units = nullptr;
  maxk::Combine* d_combine = nullptr;
  float* d_partial = nullptr;      // n_chunk_units * h floats
  unsigned* d_sched = nullptr;     // 2 x kSchedWords: forward counters, then backward counters
  int device = 0;
};

namespace maxk {

// ---------------------------------------------------------------------------------------------
// Cache-policy loads.  Streaming CSR arrays: no L1 allocation, L2 evict_first.  CBSR gathers (re-read
// ~avg_deg times, L2-resident on every 1-GPU config except products): L2 evict_last.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_keep_f32(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_keep_idx(const uint8_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_keep_idx(const uint16_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ---------------------------------------------------------------------------------------------
// Launch bookkeeping (api.cu)
// ---------------------------------------------------------------------------------------------
void note_launch(int n = 1);
int sm_count();
maxk_status_t fail(maxk_status_t s, const char* fmt, ...);
maxk_status_t check_launch(const char* what);
// Resident CTAs per SM of a kernel at (threads, dynamic smem), raising the dynamic-smem limit when needed.
// The occupancy is cached per (kernel, threads, smem, device) and the dynamic-smem limit per (kernel, device),
// only ever raised: the attribute call and occupancy query cost microseconds each,
// which launch-bound (small) graphs would otherwise pay on every layer pass.
maxk_status_t resident_ctas(const void* kern, int threads, size_t smem, const char* name, int* per_sm);

// Programmatic dependent launch (PDL, sm_90+).  The hot-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs may be scheduled while its predecessor in
// the stream is still finishing: each such kernel triggers its dependents as its CTAs start (pdl_trigger: the
// successor launches only once every CTA of this grid is resident, so it never takes a slot this grid still needs)
// and calls pdl_wait() before its first global-memory access (read or write), which returns once the predecessor
// grid has completed and its writes are visible.  Since every kernel in the chain waits before touching memory, the
// predecessor's own predecessors are complete too.  What overlaps is the launch latency, CTA rasterisation and any
// shared-memory-only prologue with the predecessor's tail.  A kernel launched without the attribute (or after a
// non-kernel stream operation) is fully serialised as usual; both instructions are then no-ops.  MAXK_PDL=0 turns
// the attribute off (A/B).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);  // errors surface through check_launch
}

// Further destinations of the top-k's CBSR rows (maxk_topk_cbsr_multi: the all-gather fused into the top-k; peers'
// replicas over NVLink or this device's): row r also goes to data[i] + r*k / idx[i] + r*k, i < n.
struct Replicas {
  int n;
  float* data[7];
  void* idx[7];
};

// launchers (return MAXK_OK or MAXK_ERR_CUDA); arguments already validated by api.cu
maxk_status_t launch_topk(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                          void* idx, cudaStream_t st);

// topk_fast_kernel with per-row probe counts (debug statistic, not the hot path)
// topk_fast_kernel writing the pair layout as well (k in {8, 16}, h in {128, 256, 384, 512}, aligned x)
maxk_status_t launch_topk_pairs(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                void* idx, uint2* pairs, cudaStream_t st, bool balanced = false);
maxk_status_t launch_topk_banked(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                 void* idx, float* bdata, void* bidx, cudaStream_t st);
maxk_status_t launch_topk_multi(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                void* idx, const Replicas& rep, cudaStream_t st);

maxk_status_t launch_topk_probe_stats(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes,
                                      float* data, void* idx, int32_t* probes, cudaStream_t st);

maxk_status_t launch_cbsr_scatter(const float* g, const void* idx, int64_t n, int h, int k, int idx_bytes, float* dx,
                                  int64_t ld, cudaStream_t st);

maxk_status_t launch_linear_topk(const void* x, int64_t n, int f_in, int64_t ldx, const void* w_t, int64_t ldw,
                                 const float* bias, int h, int k, int idx_bytes, float* data, void* idx, float* z,
                                 int64_t ldz, cudaStream_t st);

struct AggArgs {
  const int64_t* row_ptr;
  const int32_t* col;
  const float* val;
  int64_t n_rows, n_cols, nnz;
  const float* sp_data;  // fwd
  const void* sp_idx;
  int h, k;
  float* y;              // fwd out / bwd: unused
  int64_t ld_y;
  const float* dy;       // bwd in
  int64_t ld_dy;
  float* d_sp_data;      // bwd out
  // plan (units == nullptr: plan-free, one unit per row, static schedule)
  const Unit* units;
  int64_t n_units, n_chunk_units;
  float* partial;
  unsigned* sched;       // 2 counters for this kernel, or nullptr for static scheduling
  // vector kernels: units [u_short, n_units) (whole rows with <= kShortLen edges) are handed out EPI per
  // ticket, one per sub-warp; tickets run over [0, n_tix).  Set by the vector launcher.
  int64_t u_short, n_tix;
  int n_ctrs;  // ticket counters in use (1..kSchedCtrs; set by the launcher)
  int accumulate;  // 1: Y += A*CBSR (forward) / d_sp_data += ... (backward) instead of overwriting
  // forward only: the CBSR in the pair layout ({value bits, column} per entry, 8k bytes per row; maxk.h
  // maxk_spgemm_fwd_pairs) instead of sp_data / sp_idx, or nullptr
  const uint2* pairs;
  // backward only (maxk_sspmm_bwd_owners, the reduce-scatter fused into the backward): slot j's contributions go to
  // owner_dst[j / owner_rows] + (j % owner_rows) * k (device array of n_owners pointers, peers' buffers over NVLink
  // or this device's), instead of d_sp_data; nullptr otherwise
  float* const* owner_dst;
  int64_t owner_rows;
  int n_owners;
  float owner_inv;  // 1 / owner_rows (the owner is this estimate corrected by one step)
};

// Dynamic scheduling counters of one aggregation kernel: kSchedCtrs ticket counters (each on its own
// 128-byte line; warp w draws tickets w % kSchedCtrs + kSchedCtrs * n from counter w % kSchedCtrs) plus a
// done-warps counter.  One shared counter serialised ~0.9M same-address atomics per pass on
// products-shaped graphs (ncu: half the backward's stall samples on the ticket SHFL).
constexpr int kSchedCtrs = 32;
constexpr int kSchedStride = 32;                                   // unsigned words per line
constexpr int kSchedWords = (2 * kSchedCtrs + 1) * kSchedStride;   // per kernel: 2 phases + done counter

constexpr int kShortLen = 32;  // rows with at most this many edges are grouped (one batch per row)

maxk_status_t launch_spgemm_fwd(const AggArgs& a, int idx_bytes, const maxk_plan* plan, cudaStream_t st);
// vectorised kernels for k in {8,16,32,64,96,128,192,256} with aligned CBSR blocks: the forward in
// aggregate_fwd.cu (spgemm_fwd_kernel, NC = 16 replicated or NC = EPI interleaved row buffers, chosen by
// fwd_layout: h <= 256, k >= 32 and a mean degree >= 64), the backward in aggregate_bwd.cu
bool vec_path_ok(const AggArgs& a, bool fwd);
bool force_generic();
int fwd_layout(const AggArgs& a);  // 0 = NC = EPI interleaved, 1 = replicated (NC = 16; NC = 8 for k = 16 pairs)
int fwd_policy(int64_t n_rows, int64_t nnz, int h, int k, bool pairs);  // fwd_layout's decision from the sizes
maxk_status_t launch_spgemm_fwd_vec(const AggArgs& a, int idx_bytes, cudaStream_t st);
maxk_status_t launch_sspmm_bwd_vec(const AggArgs& a, int idx_bytes, cudaStream_t st);
maxk_status_t launch_sspmm_bwd(const AggArgs& a, int idx_bytes, cudaStream_t st);
maxk_status_t launch_add(float* dst, const float* src, int64_t n, cudaStream_t st);

}  // namespace maxk
