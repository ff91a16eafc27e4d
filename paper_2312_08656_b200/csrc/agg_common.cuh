// agg_common.cuh — device pieces shared by the aggregation kernels (aggregate_fwd.cu, aggregate_bwd.cu):
// the lane mapping VL<K>, vector CBSR loads, shared-memory accessors, the ticket scheduler and the launcher.
// Product code only (nothing here is shared with oracle/).
#pragma once
#include <algorithm>
#include <cstdlib>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

constexpr int VEC_THREADS = 256;

template <int K>
struct VL {
  // entries per lane per round.  (r02: 2 / 4 entries per lane at k = 8 / 16, i.e. 4 lanes and 8 edges per warp
  // step, measured within +-4% on Reddit-shaped graphs and 1.75x slower on Flickr-shaped k = 16: not kept)
  static constexpr int V = K >= 32 ? 4 : (K == 16 ? 2 : 1);
  // lanes per edge: k/V up to a warp; k = 96 / 192 (not powers of two) use 8 / 16 lanes and 3 rounds
  static constexpr int SW = K == 96 ? 8 : (K == 192 ? 16 : ((K / V) < 32 ? (K / V) : 32));
  static constexpr int EPI = 32 / SW;                          // edges per warp step
  static constexpr int R = K / (SW * V);                       // rounds per edge (K=256: 2, K=96/192: 3)
  static constexpr int U = (K >= 128 || R >= 3 || K == 8) ? 2 : 4;  // warp steps with gathers in flight
  static_assert(SW * V * R == K, "lane mapping must cover k exactly");
};

template <int V>
struct FVec;
template <>
struct FVec<1> { float v[1]; };
template <>
struct FVec<2> { float v[2]; };
template <>
struct FVec<4> { float v[4]; };

template <int V>
__device__ __forceinline__ FVec<V> ld_data(const float* p, uint64_t pol) {
  FVec<V> r;
  if constexpr (V == 4) {
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "l"(p), "l"(pol));
  } else if constexpr (V == 2) {
    asm("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(r.v[0]), "=f"(r.v[1]) : "l"(p), "l"(pol));
  } else {
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.v[0]) : "l"(p), "l"(pol));
  }
  return r;
}

// V packed indices: uint8 -> 8/16/32-bit load, uint16 -> 16/32/64-bit load.  Returned as 2 words.
template <int V, typename IdxT>
__device__ __forceinline__ uint2 ld_idx(const IdxT* p, uint64_t pol) {
  uint2 r = make_uint2(0u, 0u);
  constexpr int BYTES = V * (int)sizeof(IdxT);
  if constexpr (BYTES == 8) {
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  } else if constexpr (BYTES == 4) {
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r.x) : "l"(p), "l"(pol));
  } else if constexpr (BYTES == 2) {
    asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=r"(r.x) : "l"(p), "l"(pol));
  } else {
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(r.x) : "l"(p), "l"(pol));
  }
  return r;
}

// V entries of the pair layout ({value bits, column}, one 8- or 16-byte load: data and index come from the same
// 128-byte line in one instruction), returned as the two-block form's (data, packed index words).
template <int V, typename IdxT>
__device__ __forceinline__ void ld_pairs(const uint2* p, uint64_t pol, FVec<V>& d, uint2& x) {
  static_assert(V == 1 || V == 2, "pair layout: 1 or 2 entries per lane");
  if constexpr (V == 1) {
    uint32_t a, b;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(a), "=r"(b) : "l"(p), "l"(pol));
    d.v[0] = __uint_as_float(a);
    x = make_uint2(b, 0u);
  } else {
    uint32_t a0, b0, a1, b1;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(a0), "=r"(b0), "=r"(a1), "=r"(b1) : "l"(p), "l"(pol));
    d.v[0] = __uint_as_float(a0);
    d.v[1] = __uint_as_float(a1);
    x = make_uint2(b0 | (b1 << (8 * sizeof(IdxT))), 0u);
  }
}

template <typename IdxT>
__device__ __forceinline__ uint32_t idx_at(uint2 w, int v) {
  if constexpr (sizeof(IdxT) == 1) {
    return (w.x >> (8 * v)) & 0xffu;
  } else {
    const uint32_t word = v < 2 ? w.x : w.y;
    return (word >> (16 * (v & 1))) & 0xffffu;
  }
}

__device__ __forceinline__ float lds(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }

// Alg. 1 l.8 for one lane's R*V entries of one edge: Buf[idx] += w * data.  The entries of one CBSR row have
// distinct columns, so all loads are issued before any store (one shared-memory latency per edge step instead of
// one per entry; the asm volatile order is the program order).  STRIDE: bytes between consecutive columns.
template <int V, int R, typename IdxT, unsigned STRIDE>
__device__ __forceinline__ void rmw_entries(uint32_t buf, const uint2 (&x)[R], const FVec<V> (&d)[R], float w) {
  uint32_t adr[R][V];
  float o[R][V];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      adr[r][v] = buf + STRIDE * idx_at<IdxT>(x[r], v);
      o[r][v] = lds(adr[r][v]);
    }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int v = 0; v < V; ++v) sts(adr[r][v], fmaf(w, d[r].v[v], o[r][v]));
}

template <int V>
__device__ __forceinline__ void red_vec(float* p, const float (&g)[V]) {
  if constexpr (V == 4) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(g[0]), "f"(g[1]), "f"(g[2]), "f"(g[3])
                 : "memory");
  } else if constexpr (V == 2) {
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(g[0]), "f"(g[1]) : "memory");
  } else {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(g[0]) : "memory");
  }
}

// Dynamic LPT scheduling over degree-sorted units with n_ctrs interleaved ticket counters per phase (phase 0:
// tickets [0, u_short), the long units; phase 1: [u_short, n_tix), the grouped short rows).  Warp w draws
// tickets base + ctr + n_ctrs * m from counter ctr = w % n_ctrs; when that counter runs past the phase it
// moves on to the next counter (work stealing), and to phase 1 when every phase-0 counter is exhausted, so
// no counter's tail is left to its own warps and a warp never returns to the long units.
struct Sched {
  unsigned* sched;
  int64_t static_first, stride;
  unsigned ctr;     // counter this warp draws from (warp-uniform)
  unsigned n_ctrs;  // counters in use per phase
  int64_t u_short, n_tix;
  unsigned moves;   // counters this warp has moved past in the current phase
  int phase;
  __device__ __forceinline__ int64_t limit() const { return phase == 0 ? u_short : n_tix; }
  // lane 0 draws the next ticket of the current counter (asynchronously: resolve it later)
  __device__ __forceinline__ unsigned take(int lane) const {
    unsigned t = 0u;
    if (sched && lane == 0)
      t = (unsigned)(phase == 0 ? 0 : u_short) +
          atomicAdd(sched + (phase * kSchedCtrs + ctr) * kSchedStride, 1u) * n_ctrs + ctr;
    return t;
  }
  __device__ __forceinline__ int64_t resolve(unsigned tk, int lane) {
    int64_t t = (int64_t)__shfl_sync(FULL, tk, 0);
    while (t >= limit()) {
      if (moves + 1 < n_ctrs) {  // this counter is exhausted: steal from the next one
        ++moves;
        ctr = ctr + 1 == n_ctrs ? 0u : ctr + 1;
      } else if (phase == 0 && n_tix > u_short) {  // every long-unit counter is exhausted: grouped phase
        phase = 1;
        moves = 0;
      } else {
        return n_tix;
      }
      t = (int64_t)__shfl_sync(FULL, take(lane), 0);
    }
    return t;
  }
  __device__ __forceinline__ int64_t first(int lane) {
    if (!sched) return static_first;
    if (u_short == 0) phase = 1;
    return resolve(take(lane), lane);
  }
  __device__ __forceinline__ int64_t next(int64_t cur, unsigned tk, int lane) {
    return sched ? resolve(tk, lane) : cur + stride;
  }
  __device__ __forceinline__ void finish(int lane) const {
    if (!sched || lane != 0) return;
    const unsigned total = (gridDim.x * blockDim.x) >> 5;
    __threadfence();
    if (atomicAdd(sched + 2 * kSchedCtrs * kSchedStride, 1u) == total - 1) {  // last warp out resets counters
      for (unsigned c = 0; c < n_ctrs; ++c) {
        sched[c * kSchedStride] = 0u;
        sched[(kSchedCtrs + c) * kSchedStride] = 0u;
      }
      sched[2 * kSchedCtrs * kSchedStride] = 0u;
      __threadfence();
    }
  }
};

__device__ __forceinline__ Unit get_unit(const AggArgs& a, int64_t u) {
  if (a.units) return a.units[u];
  Unit un;
  un.row = (int32_t)u;
  un.e0 = a.row_ptr[u];
  un.len = (int32_t)(a.row_ptr[u + 1] - un.e0);
  return un;
}

template <typename Kern>
maxk_status_t launch(Kern kern, const AggArgs& a, size_t smem_per_warp, cudaStream_t st, const char* name) {
  constexpr size_t kSmemMax = 227 * 1024;
  const int warps = (int)std::min<size_t>(VEC_THREADS / 32, kSmemMax / std::max<size_t>(smem_per_warp, 1));
  if (warps < 1) return fail(MAXK_ERR_UNSUPPORTED, "%s: h=%d too large for shared memory", name, a.h);
  const int threads = warps * 32;
  const size_t smem = smem_per_warp * (size_t)warps;
  int per_sm = 0;
  const maxk_status_t s = resident_ctas(reinterpret_cast<const void*>(kern), threads, smem, name, &per_sm);
  if (s != MAXK_OK) return s;
  int64_t blocks = (int64_t)per_sm * sm_count();
  const int64_t need = (a.n_tix + warps - 1) / warps;
  if (a.sched == nullptr && blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  pdl_launch(kern, (unsigned)blocks, (unsigned)threads, smem, st, a);  // PDL (maxk_internal.cuh)
  note_launch();
  return check_launch(name);
}

// Ticket space: one ticket per long unit, one per group of EPI short units (plan only; EPI == 1 or the
// plan-free path disables grouping).
// A/B and test knob for the scheduler (unset = default).
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
// Counters per phase: ~one per 8K tickets (a warp's tail walks up to n_ctrs exhausted counters with one
// atomic each, which small graphs cannot amortise), at most kSchedCtrs.  MAXK_SCHED_CTRS overrides.
int sched_ctrs(int64_t n_tix) {
  const int forced = env_int("MAXK_SCHED_CTRS", 0);  // read per launch: tests force the stealing path
  const int64_t v = forced > 0 ? forced : n_tix / 8192;
  return (int)std::max<int64_t>(1, std::min<int64_t>(kSchedCtrs, v));
}
template <int K>
AggArgs with_tickets(const AggArgs& a0) {
  AggArgs a = a0;
  constexpr int64_t G = VL<K>::EPI;
  if (a.units == nullptr || G == 1 || a.u_short > a.n_units) a.u_short = a.n_units;
  a.n_tix = a.u_short + (a.n_units - a.u_short + G - 1) / G;
  a.n_ctrs = sched_ctrs(a.n_tix);
  return a;
}

}  // namespace
}  // namespace maxk
