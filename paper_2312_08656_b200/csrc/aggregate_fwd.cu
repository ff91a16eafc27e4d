// aggregate_fwd.cu — forward SpGEMM Y = A * densify(CBSR) (Eq. 3 left; row-wise product PAPER.md:326;
// Alg. 1) for k in {8, 16, 32, 64, 96, 128, 192, 256}.
//
// Lane mapping (agg_common.cuh VL<K>): each lane owns V consecutive CBSR entries of an edge (V = 4: one LDG.128 of
// sp_data + one LDG.32 of uint8 sp_idx, L2 evict_last), SW = k/V lanes cover an edge, a warp step covers
// EPI = 32/SW edges, U steps have their gathers in flight together; (col, val) pairs are broadcast from a
// 32-edge register batch with SHFL.  Each edge's V entries are accumulated into an on-chip row buffer (Alg. 1 l.8:
// Buf_w[sp_index[j,k]] += e_ij * sp_data[j,k]) with a non-atomic shared-memory read-modify-write — the k columns of
// one CBSR row are distinct, and a __syncwarp orders consecutive edges — and each row is written once.
//
// The read-modify-write is what bounds the forward on sm_100a (ncu r01: L1tex 99.5%, 7.77 shared wavefronts per
// edge, 66% of them bank conflicts).  A 32-lane LDS/STS of random columns c hits bank c mod 32 and costs
// max-load-of-32-balls-in-32-bins ~ 3.5 wavefronts; no static swizzle of ONE buffer helps (the selected column
// set is random), so the buffer is replicated and interleaved: copy q of column c is word NC*c + q.
//   NC = 16 (long units: rows > 32 edges and hub chunks): lane (sub-warp s, position p) accumulates into copy
//     s*CPS + p % CPS (CPS = 16/EPI), so its bank is copy + 16*(c & 1): exactly two lanes share a copy, both of
//     the SAME edge (distinct columns: no intra-instruction race), and every RMW costs 2 wavefronts.  16 KB per
//     warp at h = 256: 14 warps per SM.  At the end of a unit lane c % 32 sums the 16 copies of column c (64
//     contiguous bytes) with four LDS.128 whose quad order is rotated by lane/2 (conflict-free) and zeroes them.
//   NC = EPI: one copy per sub-warp, interleaved: the footprint of one row buffer per sub-warp (24 warps per SM)
//     with the sub-warps on disjoint banks (~3.3 wavefronts per RMW instead of ~3.5) and a contiguous end pass.
//   fwd_layout picks NC = 16 where the RMW binds (k >= 32, mean degree >= 64: Reddit- and proteins-shaped) and
//   NC = EPI where latency or the end-of-unit pass does (k <= 16, products- and Flickr-shaped), as measured.
// Pair layout (PAIRS, k in {8, 16}; maxk_spgemm_fwd_pairs): the CBSR row is k {value, column} pairs, 8k <= 128
//   bytes, so one load instruction brings both the values and the indices of an edge from ONE 128-byte line,
//   where the two blocks cost two lines (and two L1tex wavefronts) per gathered row.
// Grouped short rows (<= 32 edges, the degree-sorted tail of the plan): one row per sub-warp in the interleaved
//   single-copy layout (word EPI*c + s), pipelined across tickets; the end-of-group pass reads the EPI rows'
//   values of column c as one contiguous vector per lane and writes each row with coalesced stores.
// Scheduling: persistent CTAs; degree-sorted units by tickets from interleaved counters with work stealing
// (agg_common.cuh Sched).  Hub chunks write partial rows to plan scratch, summed in chunk order by
// combine_kernel.  Determinism: each column is summed by a fixed lane in a fixed order -> Y is bit-identical run
// to run.  Accumulating form (AggArgs::accumulate, f2 overlap): rows are added to Y instead of stored.
#include <type_traits>

#include "agg_common.cuh"

namespace maxk {
namespace {

constexpr int NC_REP = 16;  // copies of the long-unit row buffer in the replicated layout
// warp steps with gathers in flight in the NC = 16 long-unit loop (0: VL's U).  B200, Reddit-shaped, bank-balanced
// CBSR: k = 64 fwd 4.98 ms (U = 4) -> 4.69 (U = 8); k = 32 within 1% for U = 2 / 4 / 8 (tools/ab_u.sh)
#ifndef MAXK_FWD_REP_U
#define MAXK_FWD_REP_U 0
#endif
template <int K>
constexpr int rep_steps() {
  return MAXK_FWD_REP_U > 0 && VL<K>::EPI * MAXK_FWD_REP_U <= 32 ? MAXK_FWD_REP_U : (K == 64 ? 8 : VL<K>::U);
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128_zero(uint32_t a) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(a), "f"(0.0f));
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64_zero(uint32_t a) {
  asm volatile("st.shared.v2.f32 [%0], {%1,%1};" ::"r"(a), "f"(0.0f));
}

// One lane's V entries of CBSR row element offset o (= j*k + lane offset): from the two blocks (an LDG.128 of
// sp_data + an LDG.32 of sp_idx: two 128-byte lines per gathered row) or, PAIRS, from the pair layout (one
// load: k <= 16 rows are a single line).
template <int V, typename IdxT, bool PAIRS>
__device__ __forceinline__ void gather_entries(const float* dbase, const IdxT* ibase, const uint2* pbase, int64_t o,
                                               uint64_t pol, FVec<V>& d, uint2& x) {
  if constexpr (PAIRS) {
    ld_pairs<V, IdxT>(pbase + o, pol, d, x);
  } else {
    d = ld_data<V>(dbase + o, pol);
    x = ld_idx<V, IdxT>(ibase + o, pol);
  }
}

// Grouped short rows (<= 32 edges, the degree-sorted tail of the plan): one row per sub-warp in the interleaved
// single-copy layout (word EPI*c + s of the warp's region at rbase), pipelined across tickets; the end-of-group
// pass reads the EPI rows' values of column c as one contiguous vector per lane and writes each row with coalesced
// stores.  u: the warp's first ticket of this phase.  Shared by both forward layouts.
template <int K, typename IdxT, bool PAIRS>
__device__ __forceinline__ void grouped_rows(const AggArgs& a, Sched& sch, int64_t u, int lane, uint32_t rbase) {
  using L = VL<K>;
  constexpr int EPI = L::EPI, SW = L::SW, V = L::V, R = L::R, U = L::U;
  const int h = a.h;
  const int sub = lane / SW, p = lane % SW;
  const uint32_t gbuf_s = rbase + 4u * (uint32_t)sub;  // column c at + 4*EPI*c
  const float* __restrict__ dbase = a.sp_data + p * V;
  const IdxT* __restrict__ ibase = static_cast<const IdxT*>(a.sp_idx) + p * V;
  const uint2* __restrict__ pbase = a.pairs + p * V;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  constexpr int NBR = 32 / SW;  // col/val registers per lane covering a row's <= 32 edges
  struct Group {
    Unit un;
    bool have;
    int cjr[NBR];
    float cvr[NBR];
  };
  auto g_unit = [&](Group& g, int64_t t) {
    g.un.e0 = 0;
    g.un.row = 0;
    g.un.len = 0;
    g.have = false;
    if (t < a.n_tix) {
      const int64_t uq = a.u_short + (t - a.u_short) * EPI + sub;
      if (uq < a.n_units) {
        g.un = a.units[uq];
        g.have = true;
      }
    }
  };
  auto g_cols = [&](Group& g) {
#pragma unroll
    for (int i = 0; i < NBR; ++i) {
      const int e = p + i * SW;
      g.cjr[i] = 0;
      g.cvr[i] = 0.0f;
      if (e < g.un.len) {
        g.cjr[i] = ld_stream_s32(a.col + g.un.e0 + e, pol_stream);
        g.cvr[i] = ld_stream_f32(a.val + g.un.e0 + e, pol_stream);
      }
    }
  };
  auto g_proc = [&](const Group& g) {
    const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)g.un.len);
#pragma unroll
    for (int i = 0; i < NBR; ++i) {
      if (i * SW >= maxlen) break;
      for (int s0 = 0; s0 < SW && i * SW + s0 < maxlen; s0 += U) {
        FVec<V> d[U][R];
        uint2 x[U][R];
        float w[U];
        bool ok[U];
#pragma unroll
        for (int s = 0; s < U; ++s) {
          const int src = sub * SW + ((s0 + s) & (SW - 1));
          const int j = __shfl_sync(FULL, g.cjr[i], src);
          w[s] = __shfl_sync(FULL, g.cvr[i], src);
          ok[s] = (s0 + s < SW) && (i * SW + s0 + s < g.un.len);
          const int64_t o = (int64_t)j * K;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (ok[s]) {
              gather_entries<V, IdxT, PAIRS>(dbase, ibase, pbase, o + r * SW * V, pol_keep, d[s][r], x[s][r]);
            }
          }
        }
#pragma unroll
        for (int s = 0; s < U; ++s) {
          if (ok[s]) rmw_entries<V, R, IdxT, 4 * EPI>(gbuf_s, x[s], d[s], w[s]);
          __syncwarp();
        }
      }
    }
    __syncwarp();
    // end of group: lane c % 32 reads the EPI rows' values of column c (contiguous) and writes each row
    int rows[EPI];
    bool have[EPI];
#pragma unroll
    for (int s = 0; s < EPI; ++s) {
      rows[s] = __shfl_sync(FULL, g.un.row, s * SW);
      have[s] = __shfl_sync(FULL, (int)g.have, s * SW) != 0;
    }
    for (int c = lane; c < h; c += 32) {
      const uint32_t adr = rbase + (4u * EPI) * (uint32_t)c;
      float vals[EPI];
      if constexpr (EPI == 4) {
        const float4 v4 = lds128(adr);
        sts128_zero(adr);
        vals[0] = v4.x; vals[1] = v4.y; vals[2] = v4.z; vals[3] = v4.w;
      } else {
        const float2 v2 = lds64(adr);
        sts64_zero(adr);
        vals[0] = v2.x; vals[1] = v2.y;
      }
#pragma unroll
      for (int s = 0; s < EPI; ++s) {
        if (have[s]) {
          float* dst = a.y + (int64_t)rows[s] * a.ld_y + c;
          *dst = a.accumulate ? *dst + vals[s] : vals[s];
        }
      }
    }
    __syncwarp();
  };

  if (u < a.n_tix) {
    Group cur, nxt, nn;
    g_unit(cur, u);
    g_cols(cur);
    unsigned tk = sch.take(lane);
    int64_t t1 = sch.next(u, tk, lane);
    g_unit(nxt, t1);
    tk = sch.take(lane);
    while (u < a.n_tix) {
      g_cols(nxt);
      const int64_t t2 = sch.next(t1, tk, lane);
      tk = sch.take(lane);
      g_unit(nn, t2);
      g_proc(cur);
      cur = nxt;
      nxt = nn;
      u = t1;
      t1 = t2;
    }
  }
}

// NC = 16: the replicated layout above (16 KB per warp at h = 256, CTAs of up to 16 warps, 1 per SM by smem).
// NC = EPI: one copy per sub-warp, interleaved (word EPI*c + s): the same footprint as one row buffer per sub-warp
//   (4 KB per warp at h = 256, 24 warps per SM) with the sub-warps on disjoint banks (~3.3 instead of ~3.5
//   wavefronts per RMW) and a contiguous end-of-unit pass; used where occupancy matters more than conflicts.
template <int K, typename IdxT, int NC, bool PAIRS>
__global__ void __launch_bounds__(NC == NC_REP ? 512 : 256, NC == NC_REP ? 1 : 3) spgemm_fwd_kernel(const AggArgs a) {
  using L = VL<K>;
  constexpr int EPI = L::EPI, SW = L::SW, V = L::V, R = L::R;
  constexpr int U = NC == NC_REP ? rep_steps<K>() : L::U;
  constexpr int CPS = NC / EPI;  // copies per sub-warp (NC = 16: 2 lanes of the sub-warp per copy)
  static_assert(NC % EPI == 0 && SW % CPS == 0, "copy layout");
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31;
  const int h = a.h;
  const uint32_t rbase =
      (uint32_t)__cvta_generic_to_shared(reinterpret_cast<float*>(smem4) + (threadIdx.x >> 5) * (NC * h));
  const int sub = lane / SW, p = lane % SW;
  const uint32_t buf_s = rbase + 4u * (uint32_t)(sub * CPS + p % CPS);  // long units: column c at + 4*NC*c
  const float* __restrict__ dbase = a.sp_data + p * V;
  const IdxT* __restrict__ ibase = static_cast<const IdxT*>(a.sp_idx) + p * V;
  const uint2* __restrict__ pbase = a.pairs + p * V;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  // the region is zeroed once; every unit leaves it zeroed behind it (shared memory only: overlaps the
  // predecessor's tail under PDL, maxk_internal.cuh; nothing global is touched before pdl_wait)
  pdl_trigger();
  for (int w = lane; w < NC * h; w += 32) sts(rbase + 4u * w, 0.0f);
  __syncwarp();
  pdl_wait();

  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  Sched sch{a.sched, gwarp, ((int64_t)gridDim.x * blockDim.x) >> 5, (unsigned)(gwarp % a.n_ctrs),
            (unsigned)a.n_ctrs, a.u_short, a.n_tix, 0u, 0};

  // ---------------- long units ----------------
  int64_t u = sch.first(lane);
  while (u < a.n_tix && u < a.u_short) {
    const unsigned ticket = sch.take(lane);
    const Unit un = get_unit(a, u);
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
      if (eb + 32 + lane < e_end) {
        cj_n = ld_stream_s32(a.col + eb + 32 + lane, pol_stream);
        cv_n = ld_stream_f32(a.val + eb + 32 + lane, pol_stream);
      }
      // a batch whose edge weights are all equal (the SAGE mean aggregator's 1/deg row, a sum aggregator's 1)
      // skips the per-step weight SHFL: one shared-memory-pipe wavefront per warp step (ncu: ~3% of the forward)
      const float w0 = __shfl_sync(FULL, cv, 0);
      const bool uni = __all_sync(FULL, lane >= nb || __float_as_uint(cv) == __float_as_uint(w0));
      int q = 0;
      auto full_steps = [&](auto uniform) {
      for (; q + EPI * U <= nb; q += EPI * U) {  // full steps: EPI*U edges in flight, no predicates
        FVec<V> d[U][R];
        uint2 x[U][R];
        float w[U];
#pragma unroll
        for (int s = 0; s < U; ++s) {
          const int src = q + s * EPI + sub;
          const int j = __shfl_sync(FULL, cj, src);
          w[s] = decltype(uniform)::value ? w0 : __shfl_sync(FULL, cv, src);
          const int64_t o = (int64_t)j * K;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            gather_entries<V, IdxT, PAIRS>(dbase, ibase, pbase, o + r * SW * V, pol_keep, d[s][r], x[s][r]);
          }
        }
#pragma unroll
        for (int s = 0; s < U; ++s) {
          rmw_entries<V, R, IdxT, 4 * NC>(buf_s, x[s], d[s], w[s]);
          __syncwarp();  // the copy's other lane may touch this column on the next edge
        }
      }
      };
      if (uni) full_steps(std::true_type{}); else full_steps(std::false_type{});
      for (; q < nb; q += EPI) {  // batch tail: one warp step at a time, predicated per sub-warp
        const int src = q + sub;
        const int j = __shfl_sync(FULL, cj, src & 31);
        const float w = __shfl_sync(FULL, cv, src & 31);
        if (src < nb) {
          const int64_t o = (int64_t)j * K;
          FVec<V> d[R];
          uint2 x[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            gather_entries<V, IdxT, PAIRS>(dbase, ibase, pbase, o + r * SW * V, pol_keep, d[r], x[r]);
          }
          rmw_entries<V, R, IdxT, 4 * NC>(buf_s, x, d, w);
        }
        __syncwarp();
      }
      cj = cj_n;
      cv = cv_n;
    }
    __syncwarp();
    // end of unit: column c's NC copies are contiguous; lane c % 32 sums them (NC = 16: four LDS.128 whose quad
    // order is rotated by lane/2, so the 8 lanes of a quarter-warp hit 8 distinct bank quads) and zeroes them
    const bool chunk = u < a.n_chunk_units;
    float* dst = chunk ? a.partial + u * (int64_t)h : a.y + (int64_t)un.row * a.ld_y;
    const bool acc = a.accumulate && !chunk;
    for (int c = lane; c < h; c += 32) {
      float s = 0.0f;
      const uint32_t adr0 = rbase + (4u * NC) * (uint32_t)c;
      if constexpr (NC == 16) {
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t adr = adr0 + 16u * (uint32_t)((qq + (lane >> 1)) & 3);
          const float4 v4 = lds128(adr);
          sts128_zero(adr);
          s += (v4.x + v4.y) + (v4.z + v4.w);
        }
      } else if constexpr (NC == 8) {  // two LDS.128, quad order rotated by lane/4 (conflict-free quarter-warps)
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const uint32_t adr = adr0 + 16u * (uint32_t)((qq + (lane >> 2)) & 1);
          const float4 v4 = lds128(adr);
          sts128_zero(adr);
          s += (v4.x + v4.y) + (v4.z + v4.w);
        }
      } else if constexpr (NC == 4) {
        const float4 v4 = lds128(adr0);
        sts128_zero(adr0);
        s = (v4.x + v4.y) + (v4.z + v4.w);
      } else if constexpr (NC == 2) {
        const float2 v2 = lds64(adr0);
        sts64_zero(adr0);
        s = v2.x + v2.y;
      } else {
        s = lds(adr0);
        sts(adr0, 0.0f);
      }
      dst[c] = acc ? dst[c] + s : s;
    }
    __syncwarp();
    u = sch.next(u, ticket, lane);
  }

  if constexpr (EPI > 1) grouped_rows<K, IdxT, PAIRS>(a, sch, u, lane, rbase);
  sch.finish(lane);
}

// Warps per CTA for a per-warp shared-memory footprint: the CTA size (<= 16 warps) that maximises resident warps
// per SM (228 KB per SM, 227 KB per CTA, 1 KB reserved per CTA), larger CTAs on ties.
int rep_warps_per_cta(size_t smem_per_warp) {
  constexpr size_t kSmPerSm = 228 * 1024, kSmemMax = 227 * 1024, kReserved = 1024;
  int best_w = 0, best_res = 0;
  for (int w = 1; w <= 16; ++w) {
    const size_t cta = (size_t)w * smem_per_warp;
    if (cta > kSmemMax) break;
    const int ctas = (int)std::min<size_t>(kSmPerSm / (cta + kReserved), 32 / w);
    if (ctas * w >= best_res) {
      best_res = ctas * w;
      best_w = w;
    }
  }
  return best_w;
}

template <int K, typename IdxT, int NC, bool PAIRS = false>
maxk_status_t fwd_nc(const AggArgs& a0, cudaStream_t st) {
  const AggArgs a = with_tickets<K>(a0);
  auto kern = spgemm_fwd_kernel<K, IdxT, NC, PAIRS>;
  const char* name = "spgemm_fwd_kernel";
  const size_t spw = (size_t)NC * a.h * sizeof(float);
  const int rep_w = env_int("MAXK_REP_CTA_WARPS", 0);  // A/B knob: CTA size of the NC = 16 forward (0: rep_warps_per_cta)
  const int warps = NC == NC_REP ? (rep_w > 0 ? rep_w : rep_warps_per_cta(spw))
                                 : (int)std::min<size_t>(8, (227 * 1024) / spw);
  if (warps < 1) return fail(MAXK_ERR_UNSUPPORTED, "%s: h=%d too large for shared memory", name, a.h);
  const int threads = warps * 32;
  const size_t smem = spw * (size_t)warps;
  int per_sm = 0;
  const maxk_status_t s = resident_ctas(reinterpret_cast<const void*>(kern), threads, smem, name, &per_sm);
  if (s != MAXK_OK) return s;
  int64_t blocks = (int64_t)per_sm * sm_count();
  const int64_t need = (a.n_tix + warps - 1) / warps;
  if (a.sched == nullptr && blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  pdl_launch(kern, (unsigned)blocks, (unsigned)threads, smem, st, a);
  note_launch();
  return check_launch(name);
}

// layouts: 0 = NC = EPI interleaved, 1 = NC = 16 replicated
template <int K, typename IdxT, int LAYOUT>
maxk_status_t fwd_k(const AggArgs& a, cudaStream_t st) {
  return fwd_nc<K, IdxT, LAYOUT == 0 ? VL<K>::EPI : NC_REP>(a, st);
}

template <typename IdxT, int LAYOUT>
maxk_status_t nc_dispatch(const AggArgs& a, cudaStream_t st) {
  switch (a.k) {
    case 8: return fwd_k<8, IdxT, LAYOUT>(a, st);
    case 16: return fwd_k<16, IdxT, LAYOUT>(a, st);
    case 32: return fwd_k<32, IdxT, LAYOUT>(a, st);
    case 64: return fwd_k<64, IdxT, LAYOUT>(a, st);
    case 96: return fwd_k<96, IdxT, LAYOUT>(a, st);
    case 128: return fwd_k<128, IdxT, LAYOUT>(a, st);
    case 192: return fwd_k<192, IdxT, LAYOUT>(a, st);
    case 256: return fwd_k<256, IdxT, LAYOUT>(a, st);
    default: return fail(MAXK_ERR_UNSUPPORTED, "no forward kernel for k=%d", a.k);
  }
}

}  // namespace

int fwd_policy(int64_t n_rows, int64_t nnz, int h, int k, bool pairs) {
  // MAXK_FWD_REP=0 / =2 force NC = EPI / the replicated buffers (A/B and tests); default: the measured policy
  const int mode = env_int("MAXK_FWD_REP", 1);
  if (mode == 0 || h > 256) return 0;
  if (mode == 2) return 1;
  // B200, profiles/r02 (tools/ab_fwd.py): NC = 16 is faster on Reddit-shaped (mean degree 492) k = 32 / 64 and
  // proteins-shaped (299) k = 32; slower at k <= 16 (its 16 KB end-of-unit pass outweighs the saved conflicts)
  // and on products-shaped (25: latency-bound at 14 warps per SM)
  // k = 16 over the pair layout: NC = 8 on the same graphs (B200, Reddit-shaped, the mod-4-balanced pair order:
  // forward 1.82 ms with NC = EPI -> 1.77 with NC = 8; the two-block k = 16 forward keeps NC = EPI)
  const bool deg = n_rows > 0 && nnz >= 64 * n_rows;
  if (pairs) return k == 16 && deg ? 1 : 0;
  return k >= 32 && deg ? 1 : 0;
}

int fwd_layout(const AggArgs& a) { return fwd_policy(a.n_rows, a.nnz, a.h, a.k, a.pairs != nullptr); }

maxk_status_t launch_spgemm_fwd_vec(const AggArgs& a, int idx_bytes, cudaStream_t st) {
  if (a.pairs) {  // pair layout (k in {8, 16}, checked by the caller): the interleaved row buffers, as measured
    const bool b = idx_bytes == 1;
    if (a.k == 8) return b ? fwd_nc<8, uint8_t, VL<8>::EPI, true>(a, st) : fwd_nc<8, uint16_t, VL<8>::EPI, true>(a, st);
    if (a.k == 16) {  // NC = 8 row buffers (for the mod-4-balanced pair order) where the policy says so, else NC = EPI
      if (fwd_layout(a) == 0)
        return b ? fwd_nc<16, uint8_t, VL<16>::EPI, true>(a, st) : fwd_nc<16, uint16_t, VL<16>::EPI, true>(a, st);
      return b ? fwd_nc<16, uint8_t, 8, true>(a, st) : fwd_nc<16, uint16_t, 8, true>(a, st);
    }
    return fail(MAXK_ERR_UNSUPPORTED, "pair layout: k=%d not in {8, 16}", a.k);
  }
  const int layout = fwd_layout(a);
  if (idx_bytes == 1) return layout == 1 ? nc_dispatch<uint8_t, 1>(a, st) : nc_dispatch<uint8_t, 0>(a, st);
  return layout == 1 ? nc_dispatch<uint16_t, 1>(a, st) : nc_dispatch<uint16_t, 0>(a, st);
}

}  // namespace maxk
