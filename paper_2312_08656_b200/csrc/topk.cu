// topk.cu — MaxK nonlinearity -> CBSR (Eq. 1; CBSR PAPER.md:326).
//
// One warp per row; the row lives in registers (E = h/32 elements per lane).  The paper's kernel
// bisects a float pivot between min and max for "less than 10 iterations" with no
// exactness guarantee (R7).  Here:
//   phase 1 (accelerator) — probe pivots (previous row's pivot, then Illinois regula falsi on the count,
//     then bisection); a pivot with exactly k values above it makes {x > pivot} the top-k set.  Each probe
//     is one compare + predicated add per element and one warp REDUX.  ~4.5 probes on N(0,1) rows.
//   phase 2 (exact, when phase 1 cannot split exactly k: boundary ties, +-Inf, fp32 stall) — MSB-first
//     descent over order-preserving 32-bit keys to the k-th largest key, ties at it resolved toward the
//     lower column (R2); -0.0 and +0.0 share one key (R3) while the stored value keeps its bits.
// Compaction into ascending column order uses ballots, so sp_idx/sp_data are written in order.
#include <cstdlib>
#include <cstring>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

// Order-preserving key of an IEEE float (larger float -> larger key); -0.0 canonicalised to +0.0.
// Never 0 for a non-NaN input, so 0 marks padding lanes (always ranked last).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t b = __float_as_uint(f);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float key2f(uint32_t key) {
  return __uint_as_float((key & 0x80000000u) ? (key & 0x7fffffffu) : ~key);
}

// counts with one compare + one predicated add per element (the C++ form compiles to 3 instructions)
template <int E>
__device__ __forceinline__ unsigned count_gt(const float (&v)[E], float p) {
  unsigned c = 0u;
#pragma unroll
  for (int e = 0; e < E; ++e)
    asm("{\n\t.reg .pred q;\n\tsetp.gt.f32 q, %1, %2;\n\t@q add.u32 %0, %0, 1;\n\t}" : "+r"(c) : "f"(v[e]), "f"(p));
  return c;
}
template <int E>
__device__ __forceinline__ unsigned count_ge(const uint32_t (&key)[E], uint32_t t) {
  unsigned c = 0u;
#pragma unroll
  for (int e = 0; e < E; ++e)
    asm("{\n\t.reg .pred q;\n\tsetp.ge.u32 q, %1, %2;\n\t@q add.u32 %0, %0, 1;\n\t}" : "+r"(c) : "r"(key[e]), "r"(t));
  return c;
}

// predicated stores without branches
__device__ __forceinline__ void st_pred(bool p, float* a, float v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.global.f32 [%1], %2;\n\t}" ::"r"((int)p), "l"(a),
               "f"(v));
}
__device__ __forceinline__ void st_pred(bool p, uint8_t* a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.global.u8 [%1], %2;\n\t}" ::"r"((int)p), "l"(a),
               "r"(v));
}
__device__ __forceinline__ void st_pred(bool p, uint16_t* a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.global.u16 [%1], %2;\n\t}" ::"r"((int)p), "l"(a),
               "r"(v));
}

// Element e = g*G + q of lane `lane` sits at column g*32*G + lane*G + q (G = 4: float4 layout,
// G = 1: strided layout).  Column order is therefore (g, lane, q).
template <int E, int G>
__device__ __forceinline__ void prefix_in_column_order(const bool (&f)[E], int (&pos)[E], int lane) {
  const unsigned lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int g = 0; g < E / G; ++g) {
    unsigned b[G];
    int before = 0;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      b[q] = __ballot_sync(FULL, f[g * G + q]);
      before += __popc(b[q] & lt);
    }
    int own = 0;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      pos[g * G + q] = base + before + own;
      own += f[g * G + q] ? 1 : 0;
    }
#pragma unroll
    for (int q = 0; q < G; ++q) base += __popc(b[q]);
  }
}

template <int E, int G, typename IdxT>
__global__ void __launch_bounds__(256) topk_cbsr_kernel(const float* __restrict__ x, int64_t n, int h, int64_t ldx,
                                                        int k, float* __restrict__ sp_data, IdxT* __restrict__ sp_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  const int h_real = h;
  float p_prev = NAN;  // last exact pivot found by this warp (warm start for the next row)

  for (int64_t r = warp; r < n; r += nwarps) {
    const float* xr = x + r * ldx;
    float v[E];  // padding columns (scalar layout only) hold -Inf and are excluded below
#pragma unroll
    for (int g = 0; g < E / G; ++g) {
      if constexpr (G == 4) {
        const float4 f = ld_stream_f4(xr + g * 128 + lane * 4, pol);  // h % 128 == 0: no padding
        v[g * 4 + 0] = f.x; v[g * 4 + 1] = f.y; v[g * 4 + 2] = f.z; v[g * 4 + 3] = f.w;
      } else {
        const int c = g * 32 + lane;
        v[g] = c < h ? ld_stream_f32(xr + c, pol) : -INFINITY;
      }
    }
    auto is_real = [&](int e) { return G == 4 || (e * 32 + lane) < h; };

    // Phase 1 — the paper's pivot bisection used as an ACCELERATOR only: a pivot with
    // exactly k values above it makes {x > pivot} the top-k set (no tie can straddle it).  Probes: the
    // previous row's pivot, then Illinois interpolation / bisection in [min, max] (~4.5 probes on N(0,1)
    // rows).  Otherwise (ties at the boundary, +-Inf, fp32 stall, cap) fall through to the exact descent.
    bool sel[E];
    bool done = false;
    {
      float vmax = -INFINITY, vmin = INFINITY;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        vmax = fmaxf(vmax, v[e]);
        if (is_real(e)) vmin = fminf(vmin, v[e]);
      }
      // warp min/max through order-preserving keys (REDUX works on integers)
      const float hi0 = key2f(__reduce_max_sync(FULL, f2key(vmax)));
      const float lo0 = key2f(__reduce_min_sync(FULL, f2key(vmin)));
      // bracket: f(p) = count(x > p) - k; f(lo) = h - k > 0 just below the min, f(hi) = -k at the max
      float lo = nextafterf(lo0, -INFINITY), hi = hi0;
      float flo = (float)(h_real - k), fhi = -(float)k;
      // Probe order: the previous row's pivot first (rows of one layer share their value distribution),
      // then Illinois regula falsi on the count (falls back to the midpoint when interpolation stalls).
      float p = p_prev;
      int side = 0;
#pragma unroll 1
      for (int it = 0; it < 24; ++it) {
        if (!(p > lo && p < hi)) {
          p = lo + (hi - lo) * __fdividef(flo, flo - fhi);
          if (!(p > lo && p < hi)) p = 0.5f * lo + 0.5f * hi;
          if (!(p > lo && p < hi)) break;  // fp32 stall (also +-Inf endpoints): exact fallback below
        }
        const int tot = (int)__reduce_add_sync(FULL, count_gt<E>(v, p));
        if (tot == k) {
#pragma unroll
          for (int e = 0; e < E; ++e) sel[e] = v[e] > p;
          p_prev = p;
          done = true;
          break;
        }
        if (tot > k) {
          lo = p;
          flo = (float)(tot - k);
          if (side == 1) fhi *= 0.5f;  // Illinois: the retained endpoint's value is halved
          side = 1;
        } else {
          hi = p;
          fhi = (float)(tot - k);
          if (side == -1) flo *= 0.5f;
          side = -1;
        }
        p = NAN;  // next probe by interpolation
      }
    }

    // Phase 2 (exact, only when phase 1 did not split exactly k): MSB-first descent over keys,
    // T = largest key with count(key >= T) >= k (the k-th largest key).
    uint32_t T = 0u;
    bool exact = done;
    uint32_t key[E];
    if (!done) {
#pragma unroll
      for (int e = 0; e < E; ++e) key[e] = is_real(e) ? f2key(v[e]) : 0u;  // padding: key 0, ranked last
#pragma unroll 1
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cand = T | (1u << bit);
        const unsigned tot = __reduce_add_sync(FULL, count_ge<E>(key, cand));
        if (tot >= (unsigned)k) {
          T = cand;
          if (tot == (unsigned)k) { exact = true; break; }  // {key >= T} is exactly the top-k set
        }
      }
      if (exact) {
#pragma unroll
        for (int e = 0; e < E; ++e) sel[e] = key[e] >= T;
      }
    }
    if (!exact) {
      // T is the k-th largest key: take every key > T, then the lowest columns with key == T.
      unsigned gt = 0;
      bool eq[E];
#pragma unroll
      for (int e = 0; e < E; ++e) { gt += key[e] > T ? 1u : 0u; eq[e] = key[e] == T; }
      const int need = k - (int)__reduce_add_sync(FULL, gt);
      int rank[E];
      prefix_in_column_order<E, G>(eq, rank, lane);
#pragma unroll
      for (int e = 0; e < E; ++e) sel[e] = key[e] > T || (eq[e] && rank[e] < need);
    }

    int pos[E];
    prefix_in_column_order<E, G>(sel, pos, lane);
    float* drow = sp_data + r * (int64_t)k;
    IdxT* irow = sp_idx + r * (int64_t)k;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int g = e / G, q = e % G;
      const uint32_t c = (uint32_t)(g * 32 * G + lane * G + q);
      st_pred(sel[e], drow + pos[e], v[e]);
      st_pred(sel[e], irow + pos[e], c);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Newton-started probe kernel (float4 layout: h % 128 == 0, k <= 256).
//
// ncu on topk_cbsr_kernel (Reddit-shaped, k = 32): 503 issued instructions per row, issue-bound — 213 once per
// row (min/max bracket, compaction, 16 predicated scattered stores with their address arithmetic) and ~69
// per probe x 4.7 probes (the count is 18 of them; the rest is the bracket/interpolation control flow).
// Here:
//   - probe 1 at the previous row's exact pivot, probe 2 a Newton step with the previous row's local slope
//     (count per unit value); rows of one layer share their value distribution, so this usually lands on k
//     or brackets it tightly.  The [min, max] bracket is computed only when both probes fall on one side;
//   - bracketed probes use Illinois regula falsi with select-based updates and rcp.approx (probe points
//     never affect exactness: a pivot is accepted only when exactly k values exceed it);
//   - the exact MSB-first key descent is unchanged (boundary ties, +-Inf, fp32 stall);
//   - selected (value, column) pairs are compacted into a per-warp shared-memory row, then written with
//     coalesced stores (lane t writes entry t).
// Measured (B200): 493 instructions per row (probes still average ~4.8: the count is a noisy integer step
// function of the pivot, so a Newton step lands within ~2 of k, not on it); Reddit-shaped 0.136 -> 0.128 ms,
// products-shaped 1.31 -> 1.19 ms.  MAXK_TOPK_PATH=probe selects topk_cbsr_kernel (A/B).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int E, typename IdxT>
__global__ void __launch_bounds__(256) topk_newton_kernel(const float* __restrict__ x, int64_t n, int h, int64_t ldx,
                                                          int k, float* __restrict__ sp_data,
                                                          IdxT* __restrict__ sp_idx) {
  constexpr int G = 4;
  extern __shared__ uint2 stage_all[];  // k (value bits, column) pairs per warp
  uint2* stage = stage_all + (threadIdx.x >> 5) * k;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  float p_prev = NAN, s_prev = NAN;  // last exact pivot of this warp and the local count slope there

  for (int64_t r = warp; r < n; r += nwarps) {
    const float* xr = x + r * ldx;
    float v[E];
#pragma unroll
    for (int g = 0; g < E / G; ++g) {
      const float4 f = ld_stream_f4(xr + g * 128 + lane * 4, pol);
      v[g * 4 + 0] = f.x; v[g * 4 + 1] = f.y; v[g * 4 + 2] = f.z; v[g * 4 + 3] = f.w;
    }

    bool done = false;
    float p = p_prev;
    // bracket: count(x > lo) - k = flo > 0, count(x > hi) - k = fhi < 0 (infinite ends: not yet known)
    float lo = -INFINITY, hi = INFINITY, flo = 0.0f, fhi = 0.0f;
    float pa = NAN;  // the probe before p, and its count
    int ca = 0;
    if (p > -INFINITY && p < INFINITY && s_prev > 0.0f) {
      const int c1 = (int)__reduce_add_sync(FULL, count_gt<E>(v, p));
      if (c1 == k) {
        done = true;
      } else {
        if (c1 > k) { lo = p; flo = (float)(c1 - k); } else { hi = p; fhi = (float)(c1 - k); }
        pa = p;
        ca = c1;
        const float q = p + (float)(c1 - k) * rcp_approx(s_prev);  // Newton step toward count == k
        if (q > lo && q < hi) {
          p = q;
          const int c2 = (int)__reduce_add_sync(FULL, count_gt<E>(v, p));
          if (c2 == k) {
            done = true;
          } else {
            if (c2 > k) { lo = p; flo = (float)(c2 - k); } else { hi = p; fhi = (float)(c2 - k); }
            if (c2 != ca) s_prev = fabsf((float)(c2 - ca) / (p - pa));
            pa = p;
            ca = c2;
          }
        }
      }
    }
    if (!done) {
      if (!(lo > -INFINITY && hi < INFINITY)) {  // complete the bracket with the row's [min, max]
        float vmax = -INFINITY, vmin = INFINITY;
#pragma unroll
        for (int e = 0; e < E; ++e) { vmax = fmaxf(vmax, v[e]); vmin = fminf(vmin, v[e]); }
        if (!(lo > -INFINITY)) {
          lo = nextafterf(key2f(__reduce_min_sync(FULL, f2key(vmin))), -INFINITY);
          flo = (float)(h - k);
        }
        if (!(hi < INFINITY)) {
          hi = key2f(__reduce_max_sync(FULL, f2key(vmax)));
          fhi = -(float)k;
        }
      }
      int side = 0;
#pragma unroll 1
      for (int it = 0; it < 32; ++it) {
        float q = fmaf(hi - lo, flo * rcp_approx(flo - fhi), lo);
        if (!(q > lo && q < hi)) q = 0.5f * lo + 0.5f * hi;
        if (!(q > lo && q < hi)) break;  // fp32 stall (or +-Inf ends): exact descent below
        const int c = (int)__reduce_add_sync(FULL, count_gt<E>(v, q));
        if (c == k) {
          if (c != ca && pa == pa) s_prev = fabsf((float)(c - ca) / (q - pa));
          p = q;
          done = true;
          break;
        }
        if (pa == pa && c != ca) s_prev = fabsf((float)(c - ca) / (q - pa));
        pa = q;
        ca = c;
        const bool up = c > k;  // warp-uniform
        const float fc = (float)(c - k);
        fhi = up ? (side == 1 ? 0.5f * fhi : fhi) : fc;  // Illinois: halve the retained end on a repeat side
        flo = up ? fc : (side == -1 ? 0.5f * flo : flo);
        lo = up ? q : lo;
        hi = up ? hi : q;
        side = up ? 1 : -1;
      }
    }

    bool sel[E];
    if (done) {
      p_prev = p;
#pragma unroll
      for (int e = 0; e < E; ++e) sel[e] = v[e] > p;
    } else {
      // exact: T = the k-th largest key; every key > T, then the lowest columns with key == T
      uint32_t key[E];
#pragma unroll
      for (int e = 0; e < E; ++e) key[e] = f2key(v[e]);
      uint32_t T = 0u;
#pragma unroll 1
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cnd = T | (1u << bit);
        if (__reduce_add_sync(FULL, count_ge<E>(key, cnd)) >= (unsigned)k) T = cnd;
      }
      unsigned gt = 0;
      bool eq[E];
#pragma unroll
      for (int e = 0; e < E; ++e) { gt += key[e] > T ? 1u : 0u; eq[e] = key[e] == T; }
      const int need = k - (int)__reduce_add_sync(FULL, gt);
      int rank[E];
      prefix_in_column_order<E, G>(eq, rank, lane);
#pragma unroll
      for (int e = 0; e < E; ++e) sel[e] = key[e] > T || (eq[e] && rank[e] < need);
    }

    // compact (value, column) pairs into the warp's staging row in column order, then coalesced stores
    int pos[E];
    prefix_in_column_order<E, G>(sel, pos, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (sel[e]) {
        const uint32_t c = (uint32_t)((e / G) * 32 * G + lane * G + (e % G));
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(stage_s + 8u * (uint32_t)pos[e]),
                     "r"(__float_as_uint(v[e])), "r"(c));
      }
    }
    __syncwarp();
    float* drow = sp_data + r * (int64_t)k;
    IdxT* irow = sp_idx + r * (int64_t)k;
    for (int t = lane; t < k; t += 32) {
      const uint2 ent = stage[t];
      drow[t] = __uint_as_float(ent.x);
      irow[t] = (IdxT)ent.y;
    }
    __syncwarp();  // the staging row is rewritten by the next row
  }
}

template <int E, typename IdxT>
maxk_status_t run_newton(const float* x, int64_t n, int h, int64_t ldx, int k, float* data, void* idx,
                         cudaStream_t st) {
  int64_t blocks = (n + 7) / 8;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  const size_t smem = (size_t)8 * k * sizeof(uint2);
  topk_newton_kernel<E, IdxT><<<(unsigned)blocks, 256, smem, st>>>(x, n, h, ldx, k, data, (IdxT*)idx);
  note_launch();
  return check_launch("topk_newton_kernel");
}

bool probe_path_forced() {
  static const bool v = [] {
    const char* e = std::getenv("MAXK_TOPK_PATH");
    return e != nullptr && std::strcmp(e, "probe") == 0;
  }();
  return v;
}

template <int E, int G, typename IdxT>
maxk_status_t run(const float* x, int64_t n, int h, int64_t ldx, int k, float* data, void* idx, cudaStream_t st) {
  const int threads = 256;
  int64_t blocks = (n + 7) / 8;
  const int64_t cap = (int64_t)sm_count() * 16;  // oversubscribed grid measured faster than persistent
  if (blocks > cap) blocks = cap;
  topk_cbsr_kernel<E, G, IdxT><<<(unsigned)blocks, threads, 0, st>>>(x, n, h, ldx, k, data, (IdxT*)idx);
  note_launch();
  return check_launch("topk_cbsr_kernel");
}

template <typename IdxT>
maxk_status_t dispatch(const float* x, int64_t n, int h, int64_t ldx, int k, float* data, void* idx, cudaStream_t st) {
  const bool vec = (h % 128 == 0) && (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (vec && k <= 256 && !probe_path_forced()) {
    switch (h / 32) {
      case 4: return run_newton<4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 8: return run_newton<8, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 12: return run_newton<12, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 16: return run_newton<16, IdxT>(x, n, h, ldx, k, data, idx, st);
      default: break;
    }
  }
  if (vec) {
    switch (h / 32) {
      case 4: return run<4, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 8: return run<8, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 12: return run<12, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 16: return run<16, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 24: return run<24, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      case 32: return run<32, 4, IdxT>(x, n, h, ldx, k, data, idx, st);
      default: break;
    }
  }
  const int e = (h + 31) / 32;
  if (e <= 1) return run<1, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
  if (e <= 2) return run<2, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
  if (e <= 4) return run<4, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
  if (e <= 8) return run<8, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
  if (e <= 16) return run<16, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
  return run<32, 1, IdxT>(x, n, h, ldx, k, data, idx, st);
}

}  // namespace

maxk_status_t launch_topk(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                          void* idx, cudaStream_t st) {
  if (idx_bytes == 1) return dispatch<uint8_t>(x, n, h, ldx, k, data, idx, st);
  return dispatch<uint16_t>(x, n, h, ldx, k, data, idx, st);
}

}  // namespace maxk
