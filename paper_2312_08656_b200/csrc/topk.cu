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
#include "topk_row.cuh"

namespace maxk {
namespace {

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

// ------------------------------------------------------------------------------------------------
// Streamlined pivot kernel (default for h % 128 == 0, k in {8,16,32,64,96,128,192,256}; float4 layout).
//
// Same exact semantics as every path here: the selection {x > p} of a pivot p is accepted only when exactly k
// values exceed p; otherwise the exact key descent decides the row.  Per row (r02, ncu source counters on
// Reddit-shaped k = 32: 493 -> ~290 issued instructions per row, 0.118 -> 0.080 ms):
//   - warm start: probe 1 at the warp's running mean of accepted pivots, probe 2 a Newton step with the running
//     ratio of probe distance to count change; both are count-only (8 FSETP + 8 predicated adds + REDUX).  A warp
//     seeds both from its first row's moments under a Gaussian model (mean + sd * Phi^-1(1 - k/h), slope
//     sd / (h phi)): a warp handles only ~12 rows of a Reddit-shaped graph, so the seed matters;
//   - extraction: when the last probe is within 4 values of k, the missing (surplus) values are the largest
//     below (smallest above) it, found one warp max/min (REDUX on order-preserving keys) each; the resulting
//     pivot is verified by the count that the compaction computes anyway;
//   - Illinois regula falsi (rcp.approx) only for the rest (~5% of rows), bracketed lazily from the probes;
//   - compaction: per-group counts packed 8 bits each, one warp scan (5 SHFL.UP); each selected element stores
//     its value and column with two STS off one address (columns precomputed per lane), then coalesced stores;
//   - the next row of the warp is loaded while the current one is selected (register double buffer).
// STATS: the number of probes of each row is written to probes[row] (+1000 when the exact descent ran), for
// the SPEC.md:544 / PAPER.md:675 iteration statistic (maxk_topk_cbsr_probe_stats; not on the hot path).
// ------------------------------------------------------------------------------------------------
// bitmask of v[e] > p (bit e), two instructions per element (SET + LOP3)
template <int E>
__device__ __forceinline__ uint32_t mask_gt(const float (&v)[E], float p) {
  uint32_t m = 0u;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t t;
    asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(t) : "f"(v[e]), "f"(p));
    m |= t & (1u << e);
  }
  return m;
}

template <int E, int K, typename IdxT, bool STATS, bool PAIRS = false, bool BAL = false, bool MULTI = false>
#ifndef MAXK_TOPK_MINB
#define MAXK_TOPK_MINB 5  // 48 registers: 5 CTAs (40 warps) per SM; measured best against 4 (64 registers) and 6 (spills)
#endif
#ifndef MAXK_TOPK_MINB_BAL
#define MAXK_TOPK_MINB_BAL MAXK_TOPK_MINB  // the bank-balanced variants (A/B knob)
#endif
__global__ void __launch_bounds__(256, BAL ? MAXK_TOPK_MINB_BAL : MAXK_TOPK_MINB) topk_fast_kernel(const float* __restrict__ x, int64_t n, int64_t ldx,
                                                        float* __restrict__ sp_data, IdxT* __restrict__ sp_idx,
                                                        int32_t* __restrict__ probes, uint2* __restrict__ pairs,
                                                        float* __restrict__ bdata, IdxT* __restrict__ bidx,
                                                        const Replicas rep) {
  pdl_trigger();
  pdl_wait();  // PDL (maxk_internal.cuh): the previous readers of the CBSR buffers (the last backward) are complete
  constexpr int NG = E / 4;  // float4 groups per lane: element (g, q) of lane l is column 128 g + 4 l + q
  constexpr int H = 32 * E;
  static_assert(NG >= 1 && NG <= 4, "packed 8-bit group counts: at most 4 float4 groups per lane");
  // per warp: the K selected values ([0]) and columns ([1]) in column order (+ [2]: scratch of the K = 16 balanced
  // pair order)
  __shared__ uint32_t stage[PAIRS && BAL ? 3 : 2][8][K];
  const int wl = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t col[E];  // column of element e = (g, q): 128 g + 4 lane + q
#pragma unroll
  for (int e = 0; e < E; ++e) col[e] = (uint32_t)((e / 4) * 128 + lane * 4 + (e % 4));
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  PivotState ps = pivot_state(K, H);  // warm-start state of this warp's rows (topk_row.cuh)
  const uint32_t sv = (uint32_t)__cvta_generic_to_shared(&stage[0][wl][0]);
  // the next row of this warp is loaded while the current one is selected (register double buffer)
  float4 nxt[NG];
  const float* xp = x + warp * ldx + lane * 4;  // the next row to load (bumped by a pointer add per row)
  const int64_t xstep = nwarps * ldx;
  auto load_row = [&](int64_t r) {  // rows past n are not loaded (their registers are never used)
    if (r < n) {
#pragma unroll
      for (int g = 0; g < NG; ++g) nxt[g] = ld_stream_f4(xp + g * 128, pol);
    }
    xp += xstep;
  };
  load_row(warp);
  for (int64_t r = warp; r < n; r += nwarps) {
    float v[E];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      v[g * 4 + 0] = nxt[g].x; v[g * 4 + 1] = nxt[g].y; v[g * 4 + 2] = nxt[g].z; v[g * 4 + 3] = nxt[g].w;
    }
    load_row(r + nwarps);

    const int nprobe = select_row<E, STATS, sizeof(stage[0])>(v, col, K, ps, sv, lane);
    if (STATS && lane == 0) probes[r] = nprobe;
    __syncwarp();
    float* drow = sp_data + r * (int64_t)K;
    IdxT* irow = sp_idx + r * (int64_t)K;
    int n_even = 0;  // BAL: even columns among the entries already stored
    if constexpr (PAIRS && BAL && K == 16) {  // the K = 16 balanced pair order: the whole warp takes part in the votes
      const bool act = lane < K;
      float val = 0.0f;
      uint32_t c = 0u;
      if (act) {
        val = __uint_as_float(stage[0][wl][lane]);
        c = stage[1][wl][lane];
        drow[lane] = val;
        irow[lane] = (IdxT)c;
      }
      const int pos = pair16_position(c, lane, act, &stage[2][wl][0]);
      if (act) pairs[r * (int64_t)K + pos] = make_uint2(__float_as_uint(val), c);
    } else {
#pragma unroll
    for (int t0 = 0; t0 < K; t0 += 32) {
      const int t = t0 + lane;
      if (K % 32 == 0 || t < K) {
        const float val = __uint_as_float(stage[0][wl][t]);
        const uint32_t c = stage[1][wl][t];
        drow[t] = val;
        irow[t] = (IdxT)c;
        if constexpr (PAIRS) pairs[r * (int64_t)K + t] = make_uint2(__float_as_uint(val), c);  // the pair layout
        if constexpr (MULTI) {  // the all-gather fused into the top-k: the row also goes to every replica
#pragma unroll
          for (int i = 0; i < 7; ++i) {  // unrolled: constant-bank operands, no dynamic parameter indexing
            if (i < rep.n) {
              rep.data[i][r * (int64_t)K + t] = val;
              static_cast<IdxT*>(rep.idx[i])[r * (int64_t)K + t] = (IdxT)c;
            }
          }
        }
        if constexpr (BAL && !PAIRS) {  // the bank-balanced copy (K % 32 == 0): even columns from the front of Q, odd from the back
          const bool ev = (c & 1u) == 0u;
          const unsigned m = __ballot_sync(FULL, ev);
          const int ne = n_even + __popc(m & ((1u << lane) - 1u));  // even columns before t (column order)
          const int pos = bal_position(ev ? ne : K - 1 - (t - ne), K);
          n_even += __popc(m);
          bdata[r * (int64_t)K + pos] = val;
          bidx[r * (int64_t)K + pos] = (IdxT)c;
        }
      }
    }
    }
    __syncwarp();  // the staging row is rewritten by the next row
  }
}

template <int E, int K, typename IdxT, bool STATS, bool PAIRS = false, bool BAL = false, bool MULTI = false>
maxk_status_t run_fast(const float* x, int64_t n, int64_t ldx, float* data, void* idx, int32_t* probes,
                       cudaStream_t st, uint2* pairs = nullptr, float* bdata = nullptr, void* bidx = nullptr,
                       const Replicas& rep = Replicas{}) {
  int64_t blocks = (n + 7) / 8;
  static const int ctas_per_sm = [] {  // A/B knob (read once): CTAs of 8 warps per SM in the grid
    const char* e = std::getenv("MAXK_TOPK_CTAS_PER_SM");
    return e && *e ? std::atoi(e) : 16;
  }();
  const int64_t cap = (int64_t)sm_count() * ctas_per_sm;
  if (blocks > cap) blocks = cap;
  pdl_launch(topk_fast_kernel<E, K, IdxT, STATS, PAIRS, BAL, MULTI>, (unsigned)blocks, 256, 0, st, x, n, ldx, data,
             (IdxT*)idx, probes, pairs, bdata, (IdxT*)bidx, rep);
  note_launch();
  return check_launch("topk_fast_kernel");
}

// k values with a compile-time kernel (the paper's sweep); others use topk_newton_kernel
template <int E, typename IdxT, bool STATS>
maxk_status_t fast_k(const float* x, int64_t n, int64_t ldx, int k, float* data, void* idx, int32_t* probes,
                     cudaStream_t st, bool* handled) {
  *handled = true;
  switch (k) {
    case 8: return run_fast<E, 8, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    case 16: return run_fast<E, 16, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    case 32: return run_fast<E, 32, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    case 64: return run_fast<E, 64, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    case 96: return run_fast<E, 96, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    case 128: return run_fast<E, 128, IdxT, STATS>(x, n, ldx, data, idx, probes, st);
    default: *handled = false; return MAXK_OK;
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

// A/B knob (read per call): MAXK_TOPK_PATH=probe -> topk_cbsr_kernel, =newton -> topk_newton_kernel
int topk_path() {
  const char* e = std::getenv("MAXK_TOPK_PATH");
  if (e != nullptr && std::strcmp(e, "probe") == 0) return 2;
  if (e != nullptr && std::strcmp(e, "newton") == 0) return 1;
  return 0;
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
  const int path = topk_path();
  if (vec && path == 0 && h <= 512) {
    bool handled = false;
    maxk_status_t s = MAXK_OK;
    switch (h / 32) {
      case 4: s = fast_k<4, IdxT, false>(x, n, ldx, k, data, idx, nullptr, st, &handled); break;
      case 8: s = fast_k<8, IdxT, false>(x, n, ldx, k, data, idx, nullptr, st, &handled); break;
      case 12: s = fast_k<12, IdxT, false>(x, n, ldx, k, data, idx, nullptr, st, &handled); break;
      case 16: s = fast_k<16, IdxT, false>(x, n, ldx, k, data, idx, nullptr, st, &handled); break;
      default: break;
    }
    if (handled) return s;
  }
  if (vec && k <= 256 && path != 2) {
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

maxk_status_t launch_topk_probe_stats(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes,
                                      float* data, void* idx, int32_t* probes, cudaStream_t st) {
  const bool vec = (h % 128 == 0) && (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (!vec || !(h == 128 || h == 256 || h == 384 || h == 512))
    return fail(MAXK_ERR_UNSUPPORTED, "probe statistics need the float4 path (h in {128,256,384,512}, aligned x)");
  bool handled = false;
  maxk_status_t s = MAXK_OK;
  if (idx_bytes == 1) {
    switch (h / 32) {
      case 4: s = fast_k<4, uint8_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      case 8: s = fast_k<8, uint8_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      default: break;
    }
  } else {
    switch (h / 32) {
      case 4: s = fast_k<4, uint16_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      case 8: s = fast_k<8, uint16_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      case 12: s = fast_k<12, uint16_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      case 16: s = fast_k<16, uint16_t, true>(x, n, ldx, k, data, idx, probes, st, &handled); break;
      default: break;
    }
  }
  if (!handled) return fail(MAXK_ERR_UNSUPPORTED, "probe statistics: no compile-time kernel for k=%d", k);
  return s;
}

namespace {
template <int K, typename IdxT, bool BAL = false>
maxk_status_t pairs_h(const float* x, int64_t n, int h, int64_t ldx, float* data, void* idx, uint2* pairs,
                      cudaStream_t st) {
  switch (h) {
    case 128: return run_fast<4, K, IdxT, false, true, BAL>(x, n, ldx, data, idx, nullptr, st, pairs);
    case 256: return run_fast<8, K, IdxT, false, true, BAL>(x, n, ldx, data, idx, nullptr, st, pairs);
    case 384: return run_fast<12, K, IdxT, false, true, BAL>(x, n, ldx, data, idx, nullptr, st, pairs);
    case 512: return run_fast<16, K, IdxT, false, true, BAL>(x, n, ldx, data, idx, nullptr, st, pairs);
    default: return fail(MAXK_ERR_UNSUPPORTED, "pair layout: h=%d not in {128, 256, 384, 512}", h);
  }
}
}  // namespace

maxk_status_t launch_topk_pairs(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                void* idx, uint2* pairs, cudaStream_t st, bool balanced) {
  const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (!vec) return fail(MAXK_ERR_UNSUPPORTED, "pair layout: x rows must be 16-byte aligned");
  if (balanced) {
    if (k != 16) return fail(MAXK_ERR_UNSUPPORTED, "balanced pair layout: k=%d != 16", k);
    return idx_bytes == 1 ? pairs_h<16, uint8_t, true>(x, n, h, ldx, data, idx, pairs, st)
                          : pairs_h<16, uint16_t, true>(x, n, h, ldx, data, idx, pairs, st);
  }
  if (k != 8 && k != 16) return fail(MAXK_ERR_UNSUPPORTED, "pair layout: k=%d not in {8, 16}", k);
  if (idx_bytes == 1)
    return k == 8 ? pairs_h<8, uint8_t>(x, n, h, ldx, data, idx, pairs, st)
                  : pairs_h<16, uint8_t>(x, n, h, ldx, data, idx, pairs, st);
  return k == 8 ? pairs_h<8, uint16_t>(x, n, h, ldx, data, idx, pairs, st)
                : pairs_h<16, uint16_t>(x, n, h, ldx, data, idx, pairs, st);
}

namespace {
template <int K, typename IdxT>
maxk_status_t banked_h(const float* x, int64_t n, int h, int64_t ldx, float* data, void* idx, float* bdata,
                       void* bidx, cudaStream_t st) {
  switch (h) {
    case 128: return run_fast<4, K, IdxT, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, bdata, bidx);
    case 256: return run_fast<8, K, IdxT, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, bdata, bidx);
    case 384: return run_fast<12, K, IdxT, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, bdata, bidx);
    case 512: return run_fast<16, K, IdxT, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, bdata, bidx);
    default: return fail(MAXK_ERR_UNSUPPORTED, "banked order: h=%d not in {128, 256, 384, 512}", h);
  }
}
template <typename IdxT>
maxk_status_t banked_k(const float* x, int64_t n, int h, int64_t ldx, int k, float* data, void* idx, float* bdata,
                       void* bidx, cudaStream_t st) {
  switch (k) {
    case 32: return banked_h<32, IdxT>(x, n, h, ldx, data, idx, bdata, bidx, st);
    case 64: return banked_h<64, IdxT>(x, n, h, ldx, data, idx, bdata, bidx, st);
    case 128: return banked_h<128, IdxT>(x, n, h, ldx, data, idx, bdata, bidx, st);
    default: return fail(MAXK_ERR_UNSUPPORTED, "banked order: k=%d not in {32, 64, 128}", k);
  }
}
}  // namespace

maxk_status_t launch_topk_banked(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                 void* idx, float* bdata, void* bidx, cudaStream_t st) {
  const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (!vec) return fail(MAXK_ERR_UNSUPPORTED, "banked order: x rows must be 16-byte aligned");
  return idx_bytes == 1 ? banked_k<uint8_t>(x, n, h, ldx, k, data, idx, bdata, bidx, st)
                        : banked_k<uint16_t>(x, n, h, ldx, k, data, idx, bdata, bidx, st);
}

namespace {
template <int E, typename IdxT>
maxk_status_t multi_k(const float* x, int64_t n, int64_t ldx, int k, float* data, void* idx, const Replicas& rep,
                      cudaStream_t st) {
  switch (k) {
    case 8: return run_fast<E, 8, IdxT, false, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, nullptr, nullptr, rep);
    case 16: return run_fast<E, 16, IdxT, false, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, nullptr, nullptr, rep);
    case 32: return run_fast<E, 32, IdxT, false, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, nullptr, nullptr, rep);
    case 64: return run_fast<E, 64, IdxT, false, false, false, true>(x, n, ldx, data, idx, nullptr, st, nullptr, nullptr, nullptr, rep);
    default: return fail(MAXK_ERR_UNSUPPORTED, "topk multi: k=%d not in {8, 16, 32, 64}", k);
  }
}
template <typename IdxT>
maxk_status_t multi_h(const float* x, int64_t n, int h, int64_t ldx, int k, float* data, void* idx,
                      const Replicas& rep, cudaStream_t st) {
  switch (h) {
    case 128: return multi_k<4, IdxT>(x, n, ldx, k, data, idx, rep, st);
    case 256: return multi_k<8, IdxT>(x, n, ldx, k, data, idx, rep, st);
    default: return fail(MAXK_ERR_UNSUPPORTED, "topk multi: h=%d not in {128, 256}", h);
  }
}
}  // namespace

maxk_status_t launch_topk_multi(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                                void* idx, const Replicas& rep, cudaStream_t st) {
  const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (!vec) return fail(MAXK_ERR_UNSUPPORTED, "topk multi: x rows must be 16-byte aligned");
  return idx_bytes == 1 ? multi_h<uint8_t>(x, n, h, ldx, k, data, idx, rep, st)
                        : multi_h<uint16_t>(x, n, h, ldx, k, data, idx, rep, st);
}

maxk_status_t launch_topk(const float* x, int64_t n, int h, int64_t ldx, int k, int idx_bytes, float* data,
                          void* idx, cudaStream_t st) {
  if (idx_bytes == 1) return dispatch<uint8_t>(x, n, h, ldx, k, data, idx, st);
  return dispatch<uint16_t>(x, n, h, ldx, k, data, idx, st);
}

}  // namespace maxk
