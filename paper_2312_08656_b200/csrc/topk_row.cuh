// topk_row.cuh — the per-row exact top-k selection shared by the standalone MaxK kernel (topk.cu,
// topk_fast_kernel) and the fused GEMM + MaxK kernel (linear_topk.cu): Eq. 1, one warp per
// row, the row in registers (E = h/32 values per lane, element (g, q) of lane l is column 128 g + 4 l + q),
// ties to the lower column, -0.0 == +0.0 (R2, R3).  The pivot search only accelerates: a selection
// {x > p} is accepted iff exactly k values exceed p, otherwise the exact MSB-first key descent decides the row
// (R7 and §5.1).  Product code only (nothing here is shared with oracle/).
#pragma once
#include <climits>
#include <cstdint>

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

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// count of v[e] > p with one FSETP + predicated add per element
template <int E>
__device__ __forceinline__ int warp_count_gt(const float (&v)[E], float p) {
  return (int)__reduce_add_sync(FULL, count_gt<E>(v, p));
}
// bitmask helpers of the older kernels live in topk.cu
// inclusive warp scan with shfl.up's in-range predicate (2 instructions per step)
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1)
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tshfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t}"
        : "+r"(x) : "r"(d));
  return x;
}

// warp-wide extremes of the values on one side of a bound (order-preserving keys through REDUX: 4 instructions
// beyond the per-lane min/max); +-Inf when no value qualifies
template <int E>
__device__ __forceinline__ float warp_max_below(const float (&v)[E], float b) {
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < E; ++e) m = v[e] < b ? fmaxf(m, v[e]) : m;
  return key2f(__reduce_max_sync(FULL, f2key(m)));
}
template <int E>
__device__ __forceinline__ float warp_min_above(const float (&v)[E], float b) {
  float m = INFINITY;
#pragma unroll
  for (int e = 0; e < E; ++e) m = v[e] > b ? fminf(m, v[e]) : m;
  return key2f(__reduce_min_sync(FULL, f2key(m)));
}

#ifndef MAXK_TOPK_EXTRACT
#define MAXK_TOPK_EXTRACT 4  // largest |count - K| finished by extraction after the warm-start probes (0: off)
#endif
#ifndef MAXK_TOPK_DIRECT
#define MAXK_TOPK_DIRECT 2  // |count - K| after probe 1 up to which extraction follows it directly (no Newton probe)
#endif

// Bank-balanced CBSR order (include/maxk.h maxk_topk_cbsr_banked): priority rank r -> output
// position Q(r), Q = the first-half positions by group e = 0..3, then the second-half positions by group
// e = 3..0, where position 4 p + e is component e of forward lane p (L = K/8 lanes per half).  A row's even columns
// take ranks 0, 1, ... and its odd columns K-1, K-2, ...  Lanes p and p + L share an accumulator copy in the
// forward's NC = 16 layout (bank = copy + 16 (c & 1)) and conflict iff their columns have equal parity: a row with
// K/2 + d even columns has |d| same-parity pairs, in group 3 first (then 2, ...).
__device__ __forceinline__ int bal_position(int r, int K) {
  const int L = K / 8;
  if (r < K / 2) return 4 * (r % L) + r / L;
  const int q = r - K / 2;
  return 4 * (L + q % L) + 3 - q / L;
}

// Pair layout at K = 16 (include/maxk.h maxk_topk_cbsr_pairs_banked): the mod-4-balanced order read by the forward's
// NC = 8 row buffers, where lanes p = pi + 2m (m = 0..3) of entry group e share copy pi and bank = 8 (c mod 4) + ...:
// class m = c mod 4 takes lane slot m of the sets j = (e, pi) = (j >> 1, j & 1) in order j = 0, 1, 2, 3, i.e.
// position 2 (pi + 2m) + e; the entries of a class beyond its fourth (in ascending column order) fill the slots
// deficient classes leave free, ordered set 3 first, then by class.  Called by lanes 0..15 (entry t = lane in column
// order, column c); scratch: 16 words of this warp's shared memory.  Returns the position.
// Executed by the whole (converged) warp so the votes need no divergent-mask handling; lanes >= 16 pass act = false.
__device__ __forceinline__ int pair16_position(uint32_t c, int lane, bool act, uint32_t* scratch) {
  constexpr unsigned M16 = 0xffffu;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned b0 = __ballot_sync(FULL, act && (c & 1u) != 0u), b1 = __ballot_sync(FULL, act && (c & 2u) != 0u);
  const unsigned cm = ((c & 1u) ? b0 : ~b0) & ((c & 2u) ? b1 : ~b1) & M16;  // lanes of this entry's class
  const int r = __popc(cm & lt);                                              // rank within the class, column order
  // lane L < 16 stands for free-slot candidate L: set j = 3 - L / 4 (worst first), class q = L % 4; free iff n_q <= j
  const int jl = 3 - ((lane >> 2) & 3);
  const unsigned qm = ((lane & 1) ? b0 : ~b0) & ((lane & 2) ? b1 : ~b1) & M16;
  const unsigned F = __ballot_sync(FULL, act && __popc(qm) <= jl);
  const unsigned S = __ballot_sync(FULL, act && r >= 4);
  if ((F >> lane) & 1u) scratch[__popc(F & lt)] = (uint32_t)(2 * ((jl & 1) + 2 * (lane & 3)) + (jl >> 1));
  __syncwarp();
  const int own = 2 * ((r & 1) + 2 * (int)(c & 3u)) + (r >> 1);
  return r < 4 ? own : (int)scratch[__popc(S & lt) & 15];  // the s-th surplus entry takes the s-th free slot
}

// Per-warp warm-start state of the pivot search (rows of one layer share their value distribution): the running
// mean of accepted pivots, decayed sums of |dq| and |dcount| over each row's first two probes and their ratio, and
// the Gaussian-model constants of the first row's seed (zq = Phi^-1(1 - k/h), 1 / (h phi(zq))).
struct PivotState {
  float p_ref, sq, sc, rs, zq, inv_hphi;
};
__device__ __forceinline__ PivotState pivot_state(int k, int h) {
  PivotState s;
  s.zq = 1.41421356f * erfinvf(1.0f - 2.0f * (float)k / (float)h);
  s.inv_hphi = 2.50662827f * __expf(0.5f * s.zq * s.zq) / (float)h;
  s.p_ref = NAN;
  s.sq = s.sc = s.rs = 0.0f;
  return s;
}

// Select the K largest of the warp's row v (columns col) and stage them in ascending column order: values at
// shared address sv + 4 t and columns at sv + COFF + 4 t, t < K (the caller syncs the warp and stores them).
// Returns the number of probes + extraction steps (+1000 when the exact descent decided the row) if STATS.
template <int E, bool STATS, uint32_t COFF>
__device__ __forceinline__ int select_row(const float (&v)[E], const uint32_t (&col)[E], const int K, PivotState& ps,
                                          const uint32_t sv, const int lane) {
  constexpr int NG = E / 4;
  constexpr int H = 32 * E;
  static_assert(NG >= 1 && NG <= 4, "packed 8-bit group counts: at most 4 float4 groups per lane");
  // ---- pivot search (accelerator only: the final selection is accepted iff it has exactly K values) ----
  // ps.rs > 0 implies a finite ps.p_ref (the seed sets both from finite moments; updates keep them finite)
  if (!(ps.rs > 0.0f)) {  // seed from this row's moments (once per warp; again after a row with +-Inf / constant)
    float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) { s1 += v[e]; s2 = fmaf(v[e], v[e], s2); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(FULL, s1, o);
      s2 += __shfl_xor_sync(FULL, s2, o);
    }
    const float mean = s1 * (1.0f / H);
    const float sd = sqrtf(fmaxf(s2 * (1.0f / H) - mean * mean, 0.0f));
    ps.p_ref = fmaf(sd, ps.zq, mean);
    ps.rs = sd * ps.inv_hphi;
    ps.sc = 8.0f;  // prior weight of the seed slope: ~8 counts
    ps.sq = ps.rs * ps.sc;
  }
  // warm start: two count-only probes (no bracket bookkeeping: only the Illinois fallback needs it).
  // (q1, c1): the first probe; (q_last, c_last): the last one; c = -1: not probed.
  int nprobe = 0;  // probes + extraction steps (STATS only)
  const float q1 = ps.p_ref;
  const int c1 = ps.rs > 0.0f ? warp_count_gt<E>(v, q1) : -1;
  float q_last = q1;
  int c_last = c1;
  if (c1 >= 0 && (c1 - K > MAXK_TOPK_DIRECT || K - c1 > MAXK_TOPK_DIRECT)) {  // else extraction finishes directly
    const float q = fmaf((float)(c1 - K), ps.rs, q1);
    if (q > -INFINITY && q < INFINITY && q != q1) {
      const int c = warp_count_gt<E>(v, q);
      if (c != c1 && c != K) {
        ps.sq = fmaf(0.875f, ps.sq, fabsf(q - q1));
        ps.sc = fmaf(0.875f, ps.sc, (float)abs(c1 - c));
        ps.rs = ps.sq * rcp_approx(ps.sc);
      }
      q_last = q;
      c_last = c;
      if constexpr (STATS) nprobe = 1;
    }
  }
  if constexpr (STATS) nprobe += c1 >= 0 ? 1 : 0;
  bool done = c_last == K;
  float p = q_last;
#if MAXK_TOPK_EXTRACT > 0
  // finish from the last probe by extraction when it is within MAXK_TOPK_EXTRACT values of K: the m missing
  // values are the m largest at or below it (or the m surplus ones the m smallest above it), one warp max/min
  // each, in order-preserving key space.  The resulting pivot is a candidate only: it is accepted below iff
  // exactly K values exceed it (ties or +-0 at the boundary fail that check and take the exact descent).
  bool verify = false;
  if (!done && c_last >= 0 && c_last - K >= -MAXK_TOPK_EXTRACT && c_last - K <= MAXK_TOPK_EXTRACT) {
    // Positive candidates compare as their raw bits (signed int order = float order for floats >= +0): the raw
    // path saves the key conversions; a negative result (or a negative lower bound) falls back to keys.
    if (c_last < K) {
      float b = key2f(f2key(q_last) + 1u);  // v < b  <=>  v <= q_last
      bool raw = true;
#pragma unroll 1
      for (int m = c_last; m < K; ++m) {
        if (raw) {
          int mx = INT_MIN;
#pragma unroll
          for (int e = 0; e < E; ++e) mx = v[e] < b ? max(mx, __float_as_int(v[e])) : mx;
          const int t = __reduce_max_sync(FULL, mx);
          if (t >= 0) {
            b = __int_as_float(t);
            continue;
          }
          raw = false;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < E; ++e) mx = v[e] < b ? fmaxf(mx, v[e]) : mx;
        b = key2f(__reduce_max_sync(FULL, f2key(mx)));
      }
      p = key2f(f2key(b) - 1u);  // just below the K-th largest
    } else {
      float t = q_last;
      const bool raw = t >= 0.0f;  // every candidate v > t is then a positive float
#pragma unroll 1
      for (int m = c_last; m > K; --m) {
        if (raw) {
          int mn = INT_MAX;
#pragma unroll
          for (int e = 0; e < E; ++e) mn = v[e] > t ? min(mn, __float_as_int(v[e])) : mn;
          t = __int_as_float(__reduce_min_sync(FULL, mn));
        } else {
          float mn = INFINITY;
#pragma unroll
          for (int e = 0; e < E; ++e) mn = v[e] > t ? fminf(mn, v[e]) : mn;
          t = key2f(__reduce_min_sync(FULL, f2key(mn)));
        }
      }
      p = t;  // the largest value left out
    }
    if constexpr (STATS) nprobe += c_last > K ? c_last - K : K - c_last;
    done = verify = p > -INFINITY && p < INFINITY;
  }
#else
  constexpr bool verify = false;
#endif
  if (!done) {
    // Illinois regula falsi on the count, bracketed by the warm-start probes and the row's [min, max]:
    // count(x > lo) - K = flo > 0 and count(x > hi) - K = fhi < 0
    float lo = -INFINITY, hi = INFINITY, flo = (float)(H - K), fhi = -(float)K;
    auto tighten = [&](float q, int c) {
      if (c > K && q > lo) { lo = q; flo = (float)(c - K); }
      if (c >= 0 && c < K && q < hi) { hi = q; fhi = (float)(c - K); }
    };
    tighten(q1, c1);
    tighten(q_last, c_last);
    bool ok = true;
    if (!(lo > -INFINITY && hi < INFINITY)) {  // complete the bracket with the row's [min, max]
      float vmax = v[0], vmin = v[0];
#pragma unroll
      for (int e = 1; e < E; ++e) { vmax = fmaxf(vmax, v[e]); vmin = fminf(vmin, v[e]); }
      if (!(lo > -INFINITY)) {
        lo = nextafterf(key2f(__reduce_min_sync(FULL, f2key(vmin))), -INFINITY);
        flo = (float)(H - K);
      }
      if (!(hi < INFINITY)) {
        hi = key2f(__reduce_max_sync(FULL, f2key(vmax)));
        fhi = -(float)K;
      }
      ok = lo > -INFINITY && hi < INFINITY;  // +-Inf values: exact descent
    }
    // the retained end's weight is halved when the same side moves twice
    int side = 0;
#pragma unroll 1
    for (int it = 0; ok && it < 46; ++it) {
      float q = fmaf(hi - lo, flo * rcp_approx(flo - fhi), lo);
      if (!(q > lo && q < hi)) q = 0.5f * lo + 0.5f * hi;
      if (!(q > lo && q < hi)) break;  // adjacent floats: no pivot splits exactly K (ties) -> exact descent
      const int c = warp_count_gt<E>(v, q);
      if constexpr (STATS) ++nprobe;
      if (c == K) {
        p = q;
        done = true;
        break;
      }
      const int s = c > K ? 1 : -1;  // which end moved
      if (c > K) { lo = q; flo = (float)(c - K); } else { hi = q; fhi = (float)(c - K); }
      if (s == side) {
        if (s == 1) fhi *= 0.5f; else flo *= 0.5f;
      }
      side = s;
    }
  }

  // ---- selection and compaction.  sel(e): element e selected (v > p, or the exact path's mask).  Pass A
  // counts per float4 group (packed 8 bits each, <= 128 per group) for one warp scan; pass B stores each
  // selected element's value and column at its output position (two STS off one address, no register
  // shuffling).  The pivot path re-evaluates v > p in pass B instead of keeping eight predicates live. ----
  auto count_sel = [&](auto sel) {
    uint32_t packed = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) packed += sel(e) ? 1u << (8 * (e / 4)) : 0u;
    return packed;
  };
  auto place = [&](auto sel, uint32_t packed) {
    const uint32_t incl = warp_incl_scan(packed);
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    const uint32_t excl = incl - packed;
    uint32_t base = 0u;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      uint32_t adr = sv + 4u * (base + ((excl >> (8 * g)) & 0xffu));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (sel(g * 4 + q)) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(adr), "f"(v[g * 4 + q]) : "memory");
          asm volatile("st.shared.u32 [%0+%1], %2;" ::"r"(adr), "n"(COFF), "r"(col[g * 4 + q]) : "memory");
          adr += 4u;
        }
      }
      base += (tot >> (8 * g)) & 0xffu;
    }
  };
  if (done) {
    auto gt_p = [&](int e) { return v[e] > p; };
    const uint32_t packed = count_sel(gt_p);
    if (verify) {  // an extraction pivot: accepted iff exactly K values exceed it
      uint32_t c = 0u;
#pragma unroll
      for (int g = 0; g < NG; ++g) c += (packed >> (8 * g)) & 0xffu;
      done = __reduce_add_sync(FULL, c) == (uint32_t)K;
    }
    if (done) {
      ps.p_ref = fmaf(0.125f, p - ps.p_ref, ps.p_ref);
      place(gt_p, packed);
    }
  }
  if (!done) {
    // exact: T = the K-th largest key; every key > T, then the lowest columns with key == T
    uint32_t key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) key[e] = f2key(v[e]);
    uint32_t T = 0u;
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cnd = T | (1u << bit);
      if (__reduce_add_sync(FULL, count_ge<E>(key, cnd)) >= (unsigned)K) T = cnd;
    }
    unsigned gt = 0;
    bool eq[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { gt += key[e] > T ? 1u : 0u; eq[e] = key[e] == T; }
    const int need = K - (int)__reduce_add_sync(FULL, gt);
    int rank[E];
    prefix_in_column_order<E, 4>(eq, rank, lane);
    uint32_t m = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (key[e] > T || (eq[e] && rank[e] < need)) m |= 1u << e;
    auto in_m = [&](int e) { return ((m >> e) & 1u) != 0u; };
    place(in_m, count_sel(in_m));
    nprobe += 1000;
  }
  return nprobe;
}

}  // namespace
}  // namespace maxk
