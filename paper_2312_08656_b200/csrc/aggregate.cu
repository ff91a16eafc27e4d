// aggregate.cu — forward row-wise-product SpGEMM and backward outer-product SSpMM over CSR x CBSR.
//
// Forward (Eq. 3 left; Alg. 1):
//   y[i,:] = sum_{e=(i,j)} val[e] * densify(CBSR)[j,:]
//   Stage 1 (Alg. 1 l.5-9): for each edge, gather CBSR row j (k values + k indices, L2-resident) and
//   scatter-accumulate val*data into a per-(sub)warp shared-memory row buffer Buf of h floats at the
//   positions sp_idx[j,:].  Stage 2 (Alg. 1 l.12-16): ONE coalesced float4 store of the row — not the
//   paper's per-EG global atomics — because a warp owns a whole row (or a hub chunk whose partial row
//   goes to plan scratch and is summed in a fixed order by combine_kernel: deterministic).
// Backward (Eq. 3 right / Eq. 4; Alg. 2, PAPER.md:447-468, l.9 read per R8):
//   d_sp_data[j,t] += val[e] * dY[i, sp_idx[j,t]]  for every edge e=(i,j) of CSR row i.
//   Stage 1 (Alg. 2 l.3-4): coalesced float4 prefetch of dY[i,:] into the warp's shared buffer.
//   Stage 2 (Alg. 2 l.6-9): per edge, gather sp_idx[j,:], read Buf at those positions, multiply, and
//   reduce into d_sp_data[j,:] with coalesced fire-and-forget red.global.add (L2-resident target).
//
// Lane mapping (the paper's EG packing, recast): KP = k rounded up to a
// power of two.  KP <= 32: a warp step covers EPI = 32/KP edges, one per sub-warp of KP lanes, each
// sub-warp with its OWN buffer (distinct sub-warps may hit the same column).  KP > 32: one edge per
// step, EPL = KP/32 entries per lane.  Within one edge the k columns are distinct, so the non-atomic
// read-modify-write of Buf is race-free; successive edges of a sub-warp are ordered by program order.
#include <algorithm>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

constexpr int AGG_THREADS = 256;  // 8 warps per CTA
constexpr int UNROLL = 4;         // edges per sub-warp with gathers in flight together

template <int KP>
struct Lanes {
  static constexpr int SW = KP < 32 ? KP : 32;   // sub-warp width
  static constexpr int EPI = 32 / SW;             // edges per warp step
  static constexpr int EPL = KP > 32 ? KP / 32 : 1;  // entries per lane
};

// Dynamic LPT scheduling: units are sorted by decreasing cost; each warp takes the next unit from a
// global counter.  The last warp to finish resets the counters for the next launch on the stream.
struct Scheduler {
  unsigned* sched;
  int64_t static_first;
  int64_t stride;
  // lane 0 takes a ticket; the value is only broadcast (and waited for) when the unit ends
  __device__ __forceinline__ unsigned take(int lane) const {
    unsigned t = 0u;
    if (sched && lane == 0) t = atomicAdd(sched, 1u);
    return t;
  }
  __device__ __forceinline__ int64_t first(int lane) const {
    if (!sched) return static_first;
    return (int64_t)__shfl_sync(FULL, take(lane), 0);
  }
  __device__ __forceinline__ int64_t next(int64_t cur, unsigned ticket) const {
    if (!sched) return cur + stride;
    return (int64_t)__shfl_sync(FULL, ticket, 0);
  }
  __device__ __forceinline__ void finish(int lane) const {
    if (!sched || lane != 0) return;
    const unsigned total = (gridDim.x * blockDim.x) >> 5;
    __threadfence();
    const unsigned done = atomicAdd(sched + 1, 1u);
    if (done == total - 1) {  // every warp has taken its last (failing) ticket
      sched[0] = 0u;
      sched[1] = 0u;
      __threadfence();
    }
  }
};

__device__ __forceinline__ Unit load_unit(const AggArgs& a, int64_t u) {
  if (a.units) return a.units[u];
  Unit un;
  un.row = (int32_t)u;
  un.e0 = a.row_ptr[u];
  un.len = (int32_t)(a.row_ptr[u + 1] - un.e0);
  return un;
}

// ------------------------------------------------------------------------------------------------
// Forward
// ------------------------------------------------------------------------------------------------
template <int KP, typename IdxT, bool VEC>
__global__ void __launch_bounds__(AGG_THREADS) spgemm_fwd_generic_kernel(const AggArgs a) {
  using L = Lanes<KP>;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31;
  const int h = a.h, k = a.k;
  float* wbuf = smem + (threadIdx.x >> 5) * (L::EPI * h);  // this warp's EPI buffers
  const int sub = lane / L::SW, t = lane % L::SW;
  float* buf = wbuf + sub * h;
  const IdxT* __restrict__ sp_idx = static_cast<const IdxT*>(a.sp_idx);
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  for (int c = lane; c < L::EPI * h; c += 32) wbuf[c] = 0.0f;
  __syncwarp();

  const Scheduler sch{a.sched, ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                      ((int64_t)gridDim.x * blockDim.x) >> 5};
  int64_t u = sch.first(lane);
  while (u < a.n_units) {
    const unsigned ticket = sch.take(lane);  // next unit's ticket, in flight during this unit
    const Unit un = load_unit(a, u);
    const int64_t e_end = un.e0 + un.len;

    int cj = 0;
    float cv = 0.0f;
    if (un.e0 + lane < e_end) {
      cj = ld_stream_s32(a.col + un.e0 + lane, pol_stream);
      cv = ld_stream_f32(a.val + un.e0 + lane, pol_stream);
    }
    for (int64_t eb = un.e0; eb < e_end; eb += 32) {
      const int nb = (int)min((int64_t)32, e_end - eb);
      int cj_n = 0;
      float cv_n = 0.0f;
      if (eb + 32 + lane < e_end) {  // prefetch the next batch of 32 edges
        cj_n = ld_stream_s32(a.col + eb + 32 + lane, pol_stream);
        cv_n = ld_stream_f32(a.val + eb + 32 + lane, pol_stream);
      }
      for (int q = 0; q < nb; q += L::EPI * UNROLL) {
        float d[UNROLL][L::EPL];
        uint32_t x[UNROLL][L::EPL];
        float w[UNROLL];
        bool ok[UNROLL][L::EPL];
#pragma unroll
        for (int s = 0; s < UNROLL; ++s) {
          const int qe = q + s * L::EPI + sub;
          const int j = __shfl_sync(FULL, cj, qe & 31);
          w[s] = __shfl_sync(FULL, cv, qe & 31);
#pragma unroll
          for (int m = 0; m < L::EPL; ++m) {
            const int tt = t + m * 32;
            ok[s][m] = (qe < nb) && (tt < k);
            d[s][m] = 0.0f;
            x[s][m] = 0u;
            if (ok[s][m]) {
              const int64_t o = (int64_t)j * k + tt;
              d[s][m] = ld_keep_f32(a.sp_data + o, pol_keep);
              x[s][m] = ld_keep_idx(sp_idx + o, pol_keep);
            }
          }
        }
#pragma unroll
        for (int s = 0; s < UNROLL; ++s) {
#pragma unroll
          for (int m = 0; m < L::EPL; ++m)
            if (ok[s][m]) buf[x[s][m]] = fmaf(w[s], d[s][m], buf[x[s][m]]);
          __syncwarp();  // order consecutive edges' read-modify-writes (another lane may hit the same column)
        }
      }
      cj = cj_n;
      cv = cv_n;
    }
    __syncwarp();

    // Stage 2: reduce the EPI sub-warp buffers and write the row once; re-zero the buffers.
    const bool chunk = u < a.n_chunk_units;
    float* dst = chunk ? a.partial + u * (int64_t)h : a.y + (int64_t)un.row * a.ld_y;
    if (VEC) {
      for (int c = lane * 4; c < h; c += 128) {
        float4 s = *reinterpret_cast<float4*>(wbuf + c);
        *reinterpret_cast<float4*>(wbuf + c) = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = 1; b < L::EPI; ++b) {
          const float4 o = *reinterpret_cast<float4*>(wbuf + b * h + c);
          *reinterpret_cast<float4*>(wbuf + b * h + c) = make_float4(0.f, 0.f, 0.f, 0.f);
          s.x += o.x; s.y += o.y; s.z += o.z; s.w += o.w;
        }
        if (a.accumulate && !chunk) {
          const float4 o = *reinterpret_cast<const float4*>(dst + c);
          s.x += o.x; s.y += o.y; s.z += o.z; s.w += o.w;
        }
        *reinterpret_cast<float4*>(dst + c) = s;
      }
    } else {
      for (int c = lane; c < h; c += 32) {
        float s = wbuf[c];
        wbuf[c] = 0.0f;
#pragma unroll
        for (int b = 1; b < L::EPI; ++b) { s += wbuf[b * h + c]; wbuf[b * h + c] = 0.0f; }
        dst[c] = (a.accumulate && !chunk) ? dst[c] + s : s;
      }
    }
    __syncwarp();
    u = sch.next(u, ticket);
  }
  sch.finish(lane);
}

// Sum each hub row's chunk partials in chunk order (deterministic) into y (added to y when accumulating).
// VEC: float4 columns (h % 4 == 0, 16-byte aligned y rows); the chunk loads of a column are independent, the sum
// keeps chunk order.
template <bool VEC>
__global__ void __launch_bounds__(128) combine_kernel(const Combine* __restrict__ comb, const float* __restrict__ partial,
                                                      int h, float* __restrict__ y, int64_t ld_y, int accumulate) {
  pdl_trigger();
  pdl_wait();  // PDL (maxk_internal.cuh): the forward's partials are complete and visible
  const Combine cb = comb[blockIdx.x];
  float* dst = y + (int64_t)cb.row * ld_y;
  if constexpr (VEC) {
    for (int c = 4 * threadIdx.x; c < h; c += 4 * blockDim.x) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = 0; i < cb.n_chunks; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(partial + (cb.u0 + i) * (int64_t)h + c);
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      float4* d4 = reinterpret_cast<float4*>(dst + c);
      if (accumulate) {
        const float4 o = *d4;
        s.x += o.x; s.y += o.y; s.z += o.z; s.w += o.w;  // (o + s) as in the scalar form: same rounding
      }
      *d4 = s;
    }
  } else {
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      float s = 0.0f;
      for (int i = 0; i < cb.n_chunks; ++i) s += partial[(cb.u0 + i) * (int64_t)h + c];
      dst[c] = accumulate ? dst[c] + s : s;
    }
  }
}

// dst[i] += src[i] (f2: the local-target backward partial added after the overlapped reduce-scatter)
__global__ void add_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] += src[i];
}

// ------------------------------------------------------------------------------------------------
// Backward
// ------------------------------------------------------------------------------------------------
template <int KP, typename IdxT, bool VEC>
__global__ void __launch_bounds__(AGG_THREADS) sspmm_bwd_generic_kernel(const AggArgs a) {
  using L = Lanes<KP>;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31;
  const int h = a.h, k = a.k;
  float* buf = smem + (threadIdx.x >> 5) * h;  // one staged dY row per warp, read by all sub-warps
  const int sub = lane / L::SW, t = lane % L::SW;
  const IdxT* __restrict__ sp_idx = static_cast<const IdxT*>(a.sp_idx);
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  const Scheduler sch{a.sched, ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                      ((int64_t)gridDim.x * blockDim.x) >> 5};
  int64_t u = sch.first(lane);
  while (u < a.n_units) {
    const unsigned ticket = sch.take(lane);
    const Unit un = load_unit(a, u);
    if (un.len == 0) { u = sch.next(u, ticket); continue; }
    const int64_t e_end = un.e0 + un.len;

    // Stage 1: coalesced prefetch of dY[i,:] (Alg. 2 l.3-4)
    const float* src = a.dy + (int64_t)un.row * a.ld_dy;
    if (VEC) {
      for (int c = lane * 4; c < h; c += 128)
        *reinterpret_cast<float4*>(buf + c) = ld_stream_f4(src + c, pol_stream);
    } else {
      for (int c = lane; c < h; c += 32) buf[c] = ld_stream_f32(src + c, pol_stream);
    }
    int cj = 0;
    float cv = 0.0f;
    if (un.e0 + lane < e_end) {
      cj = ld_stream_s32(a.col + un.e0 + lane, pol_stream);
      cv = ld_stream_f32(a.val + un.e0 + lane, pol_stream);
    }
    __syncwarp();

    for (int64_t eb = un.e0; eb < e_end; eb += 32) {
      const int nb = (int)min((int64_t)32, e_end - eb);
      int cj_n = 0;
      float cv_n = 0.0f;
      if (eb + 32 + lane < e_end) {
        cj_n = ld_stream_s32(a.col + eb + 32 + lane, pol_stream);
        cv_n = ld_stream_f32(a.val + eb + 32 + lane, pol_stream);
      }
      for (int q = 0; q < nb; q += L::EPI * UNROLL) {
        uint32_t x[UNROLL][L::EPL];
        int j[UNROLL];
        float w[UNROLL];
        bool ok[UNROLL][L::EPL];
#pragma unroll
        for (int s = 0; s < UNROLL; ++s) {
          const int qe = q + s * L::EPI + sub;
          j[s] = __shfl_sync(FULL, cj, qe & 31);
          w[s] = __shfl_sync(FULL, cv, qe & 31);
#pragma unroll
          for (int m = 0; m < L::EPL; ++m) {
            const int tt = t + m * 32;
            ok[s][m] = (qe < nb) && (tt < k);
            x[s][m] = 0u;
            if (ok[s][m]) x[s][m] = ld_keep_idx(sp_idx + (int64_t)j[s] * k + tt, pol_keep);
          }
        }
#pragma unroll
        for (int s = 0; s < UNROLL; ++s) {
#pragma unroll
          for (int m = 0; m < L::EPL; ++m)
            if (ok[s][m]) red_add_f32(a.d_sp_data + (int64_t)j[s] * k + t + m * 32, w[s] * buf[x[s][m]]);
        }
      }
      cj = cj_n;
      cv = cv_n;
    }
    __syncwarp();  // the buffer is overwritten by the next unit's prefetch
    u = sch.next(u, ticket);
  }
  sch.finish(lane);
}

__global__ void zero4_kernel(float4* __restrict__ p4, int64_t n4, float* __restrict__ tail, int ntail) {
  pdl_trigger();
  pdl_wait();  // PDL: the previous reader of the target (the last backward) is complete
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
    p4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) tail[threadIdx.x] = 0.0f;
}

__global__ void zero1_kernel(float* __restrict__ p, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = 0.0f;
}

// ------------------------------------------------------------------------------------------------
// launch helpers
// ------------------------------------------------------------------------------------------------
// Persistent launch: CTA size = as many warps (<= 8) as the per-warp shared-memory buffers allow,
// grid = resident CTAs per SM x SM count (dynamic schedule) or just enough CTAs (static schedule).
template <typename Kern>
maxk_status_t launch_persistent(Kern kern, const AggArgs& a, size_t smem_per_warp, int64_t work_units,
                                cudaStream_t st, const char* name) {
  constexpr size_t kSmemMax = 227 * 1024;
  int warps = (int)std::min<size_t>(AGG_THREADS / 32, kSmemMax / std::max<size_t>(smem_per_warp, 1));
  if (warps < 1) return fail(MAXK_ERR_UNSUPPORTED, "%s: h=%d needs %zu B of shared memory per warp", name, a.h,
                             smem_per_warp);
  const int threads = warps * 32;
  const size_t smem = smem_per_warp * (size_t)warps;
  int per_sm = 0;
  const maxk_status_t s = resident_ctas(reinterpret_cast<const void*>(kern), threads, smem, name, &per_sm);
  if (s != MAXK_OK) return s;
  int64_t blocks = (int64_t)per_sm * sm_count();
  const int64_t need = (work_units + warps - 1) / warps;
  if (a.sched == nullptr && blocks > need) blocks = need;  // static schedule: no idle warps needed
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, threads, smem, st>>>(a);
  note_launch();
  return check_launch(name);
}

template <int KP, typename IdxT>
maxk_status_t fwd_k(const AggArgs& a, cudaStream_t st) {
  const bool vec = (a.h % 4 == 0) && (a.ld_y % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15u) == 0);
  const size_t smem = (size_t)Lanes<KP>::EPI * a.h * sizeof(float);
  if (vec) return launch_persistent(spgemm_fwd_generic_kernel<KP, IdxT, true>, a, smem, a.n_units, st, "spgemm_fwd_generic_kernel");
  return launch_persistent(spgemm_fwd_generic_kernel<KP, IdxT, false>, a, smem, a.n_units, st, "spgemm_fwd_generic_kernel");
}

template <int KP, typename IdxT>
maxk_status_t bwd_k(const AggArgs& a, cudaStream_t st) {
  const bool vec = (a.h % 4 == 0) && (a.ld_dy % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.dy) & 15u) == 0);
  const size_t smem = (size_t)a.h * sizeof(float);
  if (vec) return launch_persistent(sspmm_bwd_generic_kernel<KP, IdxT, true>, a, smem, a.n_units, st, "sspmm_bwd_generic_kernel");
  return launch_persistent(sspmm_bwd_generic_kernel<KP, IdxT, false>, a, smem, a.n_units, st, "sspmm_bwd_generic_kernel");
}

template <typename IdxT>
maxk_status_t fwd_dispatch(const AggArgs& a, cudaStream_t st) {
  const int k = a.k;
  if (k <= 4) return fwd_k<4, IdxT>(a, st);  // sub-warps of >= 4 lanes: <= 8 row buffers per warp
  if (k <= 8) return fwd_k<8, IdxT>(a, st);
  if (k <= 16) return fwd_k<16, IdxT>(a, st);
  if (k <= 32) return fwd_k<32, IdxT>(a, st);
  if (k <= 64) return fwd_k<64, IdxT>(a, st);
  if (k <= 128) return fwd_k<128, IdxT>(a, st);
  if (k <= 256) return fwd_k<256, IdxT>(a, st);
  if (k <= 512) return fwd_k<512, IdxT>(a, st);
  if (k <= 1024) return fwd_k<1024, IdxT>(a, st);
  return fail(MAXK_ERR_UNSUPPORTED, "k=%d > 1024 not supported by this build", k);
}

template <typename IdxT>
maxk_status_t bwd_dispatch(const AggArgs& a, cudaStream_t st) {
  const int k = a.k;
  if (k <= 4) return bwd_k<4, IdxT>(a, st);  // sub-warps of >= 4 lanes: <= 8 row buffers per warp
  if (k <= 8) return bwd_k<8, IdxT>(a, st);
  if (k <= 16) return bwd_k<16, IdxT>(a, st);
  if (k <= 32) return bwd_k<32, IdxT>(a, st);
  if (k <= 64) return bwd_k<64, IdxT>(a, st);
  if (k <= 128) return bwd_k<128, IdxT>(a, st);
  if (k <= 256) return bwd_k<256, IdxT>(a, st);
  if (k <= 512) return bwd_k<512, IdxT>(a, st);
  if (k <= 1024) return bwd_k<1024, IdxT>(a, st);
  return fail(MAXK_ERR_UNSUPPORTED, "k=%d > 1024 not supported by this build", k);
}

maxk_status_t zero_fill(float* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return MAXK_OK;
  const int64_t cap = (int64_t)sm_count() * 8;
  if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
    const int64_t n4 = n / 4;
    int64_t blocks = (n4 + 255) / 256;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    pdl_launch(zero4_kernel, (unsigned)blocks, 256, 0, st, reinterpret_cast<float4*>(p), n4, p + n4 * 4,
               (int)(n - n4 * 4));
  } else {
    int64_t blocks = (n + 255) / 256;
    if (blocks > cap) blocks = cap;
    zero1_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, n);
  }
  note_launch();
  return check_launch("zero_kernel");
}

}  // namespace

maxk_status_t launch_spgemm_fwd(const AggArgs& a, int idx_bytes, const maxk_plan* plan, cudaStream_t st) {
  if (a.n_units > 0) {
    maxk_status_t s;
    if (a.pairs || (!force_generic() && vec_path_ok(a, true)))  // the pair layout exists only on the vector path
      s = launch_spgemm_fwd_vec(a, idx_bytes, st);
    else
      s = idx_bytes == 1 ? fwd_dispatch<uint8_t>(a, st) : fwd_dispatch<uint16_t>(a, st);
    if (s != MAXK_OK) return s;
  }
  if (plan && plan->n_split_rows > 0) {
    const bool vec = a.h % 4 == 0 && a.ld_y % 4 == 0 && (reinterpret_cast<uintptr_t>(a.y) & 15u) == 0;
    pdl_launch(vec ? combine_kernel<true> : combine_kernel<false>, (unsigned)plan->n_split_rows,
               vec ? 64u : 128u, 0, st, (const Combine*)plan->d_combine, (const float*)plan->d_partial, a.h, a.y,
               a.ld_y, a.accumulate);
    note_launch();
    return check_launch("combine_kernel");
  }
  return MAXK_OK;
}

maxk_status_t launch_sspmm_bwd(const AggArgs& a, int idx_bytes, cudaStream_t st) {
  if (!a.accumulate) {
    maxk_status_t s = zero_fill(a.d_sp_data, a.n_cols * (int64_t)a.k, st);
    if (s != MAXK_OK) return s;
  }
  if (a.n_units == 0) return MAXK_OK;
  if (!force_generic() && vec_path_ok(a, false)) return launch_sspmm_bwd_vec(a, idx_bytes, st);
  return idx_bytes == 1 ? bwd_dispatch<uint8_t>(a, st) : bwd_dispatch<uint16_t>(a, st);
}

maxk_status_t launch_add(float* dst, const float* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return MAXK_OK;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  add_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, src, n);
  note_launch();
  return check_launch("add_kernel");
}

}  // namespace maxk
