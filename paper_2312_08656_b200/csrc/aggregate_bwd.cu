// aggregate_bwd.cu — vectorised backward SSpMM for k in {8, 16, 32, 64, 96, 128, 192, 256} (Alg. 2, PAPER.md:447-468;
// Eq. 3 right and Eq. 4; line 9 read as d_sp_data[j,t] += A[i,j] * dY[i, sp_idx[j,t]], R8).
//
// Lane mapping as the forward (agg_common.cuh VL<K>): each lane owns V consecutive CBSR entries of an edge (one
// LDG of V indices), SW = k/V lanes cover an edge, a warp step covers EPI = 32/SW edges; (col, val) pairs are
// broadcast from a 32-edge register batch with SHFL.  Stage 1 (Alg. 2 l.1-5) stages the dense row dY[i,:] into
// shared memory once per unit (read-only); stage 2 (l.6-9) gathers it at the CBSR indices of each edge's column
// j and reduces the V products into d_sp_data[j] with one 16-byte red.global.add.v4.f32 per lane (fire and forget,
// merged in L2, where the 30 MB d_sp_data of Reddit-shaped graphs stays resident).
// Scheduling: persistent CTAs; degree-sorted units handed out by tickets from interleaved counters with work
// stealing (agg_common.cuh Sched); rows of <= 32 edges are grouped EPI per ticket.
// Accumulating form (AggArgs::accumulate, f2 overlap): the zero-fill of d_sp_data is skipped (launch_sspmm_bwd).
#include <type_traits>

#include "agg_common.cuh"

namespace maxk {
namespace {

// ------------------------------------------------------------------------------------------------
// Backward
// ------------------------------------------------------------------------------------------------
template <int K, typename IdxT, bool VEC_DY, bool OWN = false>
__global__ void __launch_bounds__(VEC_THREADS) sspmm_bwd_vec_kernel(const AggArgs a) {
  pdl_trigger();
  pdl_wait();  // PDL (maxk_internal.cuh): the CBSR indices and the zeroed target are complete and visible
  using L = VL<K>;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31;
  const int h = a.h;
  float* wbuf = smem + (threadIdx.x >> 5) * (L::EPI * h);  // EPI buffers: grouped short rows use one each
  float* buf = wbuf;                                        // a long unit's staged row, shared by sub-warps
  const int sub = lane / L::SW, p = lane % L::SW;
  const uint32_t buf_s = (uint32_t)__cvta_generic_to_shared(buf);
  const IdxT* __restrict__ ibase = static_cast<const IdxT*>(a.sp_idx) + p * L::V;
  float* __restrict__ obase = a.d_sp_data + p * L::V;
  // reduction target of CBSR row (slot) j: this call's d_sp_data, or (OWN: the reduce-scatter fused into the
  // backward) row j % owner_rows of the owner's block, owner j / owner_rows, written over peer memory
  auto target = [&](int j) -> float* {
    if constexpr (OWN) {
      uint32_t g = __float2uint_rz(__uint2float_rz((uint32_t)j) * a.owner_inv);
      if ((int64_t)(g + 1) * a.owner_rows <= j) ++g;
      if ((int64_t)g * a.owner_rows > j) --g;
      return a.owner_dst[g] + p * L::V + ((int64_t)j - (int64_t)g * a.owner_rows) * K;
    } else {
      return obase + (int64_t)j * K;
    }
  };
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  Sched sch{a.sched, gwarp, ((int64_t)gridDim.x * blockDim.x) >> 5, (unsigned)(gwarp % a.n_ctrs),
            (unsigned)a.n_ctrs, a.u_short, a.n_tix, 0u, 0};

  // ---- grouped short rows (<= 32 edges): one row per sub-warp, each staging its own dY row into its own
  // buffer (a double-buffered cp.async prefetch of the next ticket's rows was measured no faster). ----
  constexpr int NBR = 32 / L::SW;
  struct Group {
    Unit un;
    int cjr[NBR];
    float cvr[NBR];
  };
  auto g_unit = [&](Group& g, int64_t t) {
    g.un.e0 = 0;
    g.un.row = 0;
    g.un.len = 0;
    if (t < a.n_tix) {
      const int64_t uq = a.u_short + (t - a.u_short) * L::EPI + sub;
      if (uq < a.n_units) g.un = a.units[uq];
    }
  };
  auto g_cols = [&](Group& g) {
#pragma unroll
    for (int i = 0; i < NBR; ++i) {
      const int e = p + i * L::SW;
      g.cjr[i] = 0;
      g.cvr[i] = 0.0f;
      if (e < g.un.len) {
        g.cjr[i] = ld_stream_s32(a.col + g.un.e0 + e, pol_stream);
        g.cvr[i] = ld_stream_f32(a.val + g.un.e0 + e, pol_stream);
      }
    }
  };
  auto g_stage = [&](const Group& g) {
    float* mybuf = wbuf + sub * h;
    if (g.un.len == 0) return;
    const float* src_row = a.dy + (int64_t)g.un.row * a.ld_dy;
    if (VEC_DY) {
      for (int c = p * 4; c < h; c += L::SW * 4)
        *reinterpret_cast<float4*>(mybuf + c) = ld_stream_f4(src_row + c, pol_stream);
    } else {
      for (int c = p; c < h; c += L::SW) mybuf[c] = ld_stream_f32(src_row + c, pol_stream);
    }
  };
  auto g_proc = [&](const Group& g) {
    const uint32_t my_s = (uint32_t)__cvta_generic_to_shared(wbuf + sub * h);
    const int maxlen = (int)__reduce_max_sync(FULL, (unsigned)g.un.len);
#pragma unroll
    for (int i = 0; i < NBR; ++i) {
      if (i * L::SW >= maxlen) break;
      for (int s0 = 0; s0 < L::SW && i * L::SW + s0 < maxlen; s0 += L::U) {
        uint2 x[L::U][L::R];
        int64_t o[L::U];
        float w[L::U];
        bool ok[L::U];
        int jj[L::U];
#pragma unroll
        for (int s = 0; s < L::U; ++s) {
          const int src = sub * L::SW + ((s0 + s) & (L::SW - 1));
          const int j = __shfl_sync(FULL, g.cjr[i], src);
          jj[s] = j;
          w[s] = __shfl_sync(FULL, g.cvr[i], src);
          ok[s] = (s0 + s < L::SW) && (i * L::SW + s0 + s < g.un.len);
          o[s] = (int64_t)j * K;
#pragma unroll
          for (int r = 0; r < L::R; ++r)
            if (ok[s]) x[s][r] = ld_idx<L::V, IdxT>(ibase + o[s] + r * L::SW * L::V, pol_keep);
        }
#pragma unroll
        for (int s = 0; s < L::U; ++s) {
          if (ok[s]) {
#pragma unroll
            for (int r = 0; r < L::R; ++r) {
              float gv[L::V];
#pragma unroll
              for (int v = 0; v < L::V; ++v) gv[v] = w[s] * lds(my_s + 4u * idx_at<IdxT>(x[s][r], v));
              red_vec<L::V>(target(jj[s]) + r * L::SW * L::V, gv);
            }
          }
        }
      }
    }
  };

  int64_t u = sch.first(lane);
  while (u < a.n_tix && u < a.u_short) {  // ---- long units (whole rows > 32 edges, hub chunks) ----
    const unsigned ticket = sch.take(lane);
    const Unit un = get_unit(a, u);
    if (un.len == 0) {
      u = sch.next(u, ticket, lane);
      continue;
    }
    const int64_t e_end = un.e0 + un.len;
    const float* src_row = a.dy + (int64_t)un.row * a.ld_dy;
    if (VEC_DY) {
      for (int c = lane * 4; c < h; c += 128)
        *reinterpret_cast<float4*>(buf + c) = ld_stream_f4(src_row + c, pol_stream);
    } else {
      for (int c = lane; c < h; c += 32) buf[c] = ld_stream_f32(src_row + c, pol_stream);
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
      // a batch whose edge weights are all equal skips the per-step weight SHFL (aggregate_fwd.cu)
      const float w0 = __shfl_sync(FULL, cv, 0);
      const bool uni = __all_sync(FULL, lane >= nb || __float_as_uint(cv) == __float_as_uint(w0));
      int q = 0;
      auto full_steps = [&](auto uniform) {
      for (; q + L::EPI * L::U <= nb; q += L::EPI * L::U) {
        uint2 x[L::U][L::R];
        int64_t o[L::U];
        float w[L::U];
        int jj[L::U];
#pragma unroll
        for (int s = 0; s < L::U; ++s) {
          const int src = q + s * L::EPI + sub;
          const int j = __shfl_sync(FULL, cj, src);
          jj[s] = j;
          w[s] = decltype(uniform)::value ? w0 : __shfl_sync(FULL, cv, src);
          o[s] = (int64_t)j * K;
#pragma unroll
          for (int r = 0; r < L::R; ++r) x[s][r] = ld_idx<L::V, IdxT>(ibase + o[s] + r * L::SW * L::V, pol_keep);
        }
#pragma unroll
        for (int s = 0; s < L::U; ++s)
#pragma unroll
          for (int r = 0; r < L::R; ++r) {
            float g[L::V];
#pragma unroll
            for (int v = 0; v < L::V; ++v) g[v] = w[s] * lds(buf_s + 4u * idx_at<IdxT>(x[s][r], v));
            red_vec<L::V>(target(jj[s]) + r * L::SW * L::V, g);
          }
      }
      };
      if (uni) full_steps(std::true_type{}); else full_steps(std::false_type{});
      for (; q < nb; q += L::EPI) {
        const int src = q + sub;
        const bool ok = src < nb;
        const int j = __shfl_sync(FULL, cj, src & 31);
        const float w = __shfl_sync(FULL, cv, src & 31);
        if (ok) {
          const int64_t o = (int64_t)j * K;
#pragma unroll
          for (int r = 0; r < L::R; ++r) {
            const uint2 x = ld_idx<L::V, IdxT>(ibase + o + r * L::SW * L::V, pol_keep);
            float g[L::V];
#pragma unroll
            for (int v = 0; v < L::V; ++v) g[v] = w * lds(buf_s + 4u * idx_at<IdxT>(x, v));
            red_vec<L::V>(target(j) + r * L::SW * L::V, g);
          }
        }
      }
      cj = cj_n;
      cv = cv_n;
    }
    __syncwarp();
    u = sch.next(u, ticket, lane);
  }
  while (u < a.n_tix) {  // ---- grouped phase ----
    const unsigned ticket = sch.take(lane);
    Group cur;
    g_unit(cur, u);
    g_cols(cur);
    g_stage(cur);
    __syncwarp();
    g_proc(cur);
    __syncwarp();  // the buffers are overwritten by the next ticket's staging
    u = sch.next(u, ticket, lane);
  }
  sch.finish(lane);
}

template <int K, typename IdxT>
maxk_status_t bwd_vec(const AggArgs& a0, cudaStream_t st) {
  const AggArgs a = with_tickets<K>(a0);
  const bool vd = (a.h % 4 == 0) && (a.ld_dy % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.dy) & 15u) == 0);
  const size_t smem = (size_t)VL<K>::EPI * a.h * sizeof(float);
  if (a.owner_dst != nullptr) {
    if (vd) return launch(sspmm_bwd_vec_kernel<K, IdxT, true, true>, a, smem, st, "sspmm_bwd_vec_kernel");
    return launch(sspmm_bwd_vec_kernel<K, IdxT, false, true>, a, smem, st, "sspmm_bwd_vec_kernel");
  }
  if (vd) return launch(sspmm_bwd_vec_kernel<K, IdxT, true>, a, smem, st, "sspmm_bwd_vec_kernel");
  return launch(sspmm_bwd_vec_kernel<K, IdxT, false>, a, smem, st, "sspmm_bwd_vec_kernel");
}

template <typename IdxT>
maxk_status_t dispatch(const AggArgs& a, cudaStream_t st) {
  switch (a.k) {
    case 8: return bwd_vec<8, IdxT>(a, st);
    case 16: return bwd_vec<16, IdxT>(a, st);
    case 32: return bwd_vec<32, IdxT>(a, st);
    case 64: return bwd_vec<64, IdxT>(a, st);
    case 96: return bwd_vec<96, IdxT>(a, st);
    case 128: return bwd_vec<128, IdxT>(a, st);
    case 192: return bwd_vec<192, IdxT>(a, st);
    case 256: return bwd_vec<256, IdxT>(a, st);
    default: return fail(MAXK_ERR_UNSUPPORTED, "no vector kernel for k=%d", a.k);
  }
}

}  // namespace

bool vec_path_ok(const AggArgs& a, bool fwd) {
  const int k = a.k;
  if (k != 8 && k != 16 && k != 32 && k != 64 && k != 96 && k != 128 && k != 192 && k != 256) return false;
  // V-wide loads of sp_data / sp_idx rows need their natural alignment
  const uintptr_t ip = reinterpret_cast<uintptr_t>(a.sp_idx);
  if (fwd && (reinterpret_cast<uintptr_t>(a.sp_data) & 15u) != 0) return false;
  if (!fwd && (reinterpret_cast<uintptr_t>(a.d_sp_data) & 15u) != 0) return false;
  return (ip & 7u) == 0;
}

maxk_status_t launch_sspmm_bwd_vec(const AggArgs& a, int idx_bytes, cudaStream_t st) {
  return idx_bytes == 1 ? dispatch<uint8_t>(a, st) : dispatch<uint16_t>(a, st);
}

}  // namespace maxk
