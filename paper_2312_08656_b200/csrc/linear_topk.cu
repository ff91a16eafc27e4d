// linear_topk.cu — Eq. 1 fused: h(X) = max-k (X·W + b) -> CBSR.
//
// One persistent CTA per SM, warp-specialised (sm_100a tcgen05 / TMEM / TMA):
//   warp 0      TMA producer: loads W^T once (resident in shared memory, 128B-swizzled K-major), then streams
//               128 x 64 bf16 tiles of X through a STAGES-deep mbarrier ring;
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32,
//               M=128, N=h, K=16) into a double-buffered TMEM accumulator (2 x h columns);
//   warps 2..9  epilogue: thread-per-row — TMEM lane r is row r of the tile, read 32 columns at a time with
//               tcgen05.ld.32x32b.x32; z = acc + b; exact top-k of the row's h values of z (pivot probes with
//               Illinois interpolation and a warm start from the thread's previous row; exact MSB-first key
//               descent when no pivot splits exactly k), emitted in ascending column order straight to
//               sp_data / sp_idx.  Two groups of 4 warps take alternate tiles (one TMEM accumulator stage each),
//               so two tiles' epilogues run while the tensor cores fill the next accumulator.
// The selection is the exact top-k of the fp32 z the kernel computes (ties -> lower column, -0 == +0),
// identical to maxk_topk_cbsr applied to z; z itself can be written out (z_out) for verification.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

constexpr int BM = 128;          // rows per tile (UMMA M)
constexpr int BK = 64;           // bf16 elements per 128-byte swizzle row (one k-block)
constexpr int STAGES = 3;        // X tile ring depth
constexpr int EPI_WARPS = 8;  // two groups of 4 (one per TMEM accumulator stage / TMEM lane quarter)
constexpr int THREADS = (2 + EPI_WARPS) * 32;

struct __align__(8) Barriers {
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2], wbar;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
// try_wait with a suspend-time hint (ns): the producer / MMA threads are parked until the phase flips instead of
// spinning and taking issue slots from the epilogue warps on the same scheduler
__device__ __forceinline__ void mbar_wait_parked(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(s32(b)),
      "r"(parity), "r"(20000u)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          s32(dst)),
      "l"(map), "r"(s32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte-swizzled shared-memory matrix descriptor (cute::UMMA::SmemDescriptor layout):
// start address >>4 in [0,14), LBO (ignored for SW128 K-major) = 1, SBO = 1024 B (8 rows x 128 B) >>4 in
// [32,46), version 1 in [46,48), layout SWIZZLE_128B = 2 in [61,64).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor (cute::UMMA::InstrDescriptor): c_format F32 (bit 4), a/b format BF16 (bits 7, 10),
// K-major A and B, N >> 3 in [17,23), M >> 4 in [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t b = __float_as_uint(f);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// one pass over the thread's row: f(j, c, z) with z[c] = acc[c] + bias[c] for c in [0, H), chunk by chunk from
// TMEM; j = c mod 32 is a compile-time constant after unrolling (used to spread accumulators for ILP)
template <int H, typename F>
__device__ __forceinline__ void row_pass(uint32_t taddr, F&& f) {
#pragma unroll 1
  for (int c0 = 0; c0 < H; c0 += 64) {  // two 32-column TMEM loads in flight per wait
    uint32_t r[32], r2[32];
    tmem_ld32(taddr + (uint32_t)c0, r);
    tmem_ld32(taddr + (uint32_t)c0 + 32u, r2);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) f(j, c0 + j, __uint_as_float(r[j]));
#pragma unroll
    for (int j = 0; j < 32; ++j) f(j, c0 + 32 + j, __uint_as_float(r2[j]));
  }
}
// pass 0: z = acc + bias, written back into the accumulator's TMEM columns (later passes read z directly)
template <int H, typename F>
__device__ __forceinline__ void bias_pass(uint32_t taddr, const float* bias_s, F&& f) {
#pragma unroll 1
  for (int c0 = 0; c0 < H; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + (uint32_t)c0, r);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float z = __uint_as_float(r[j]) + bias_s[c0 + j];
      f(j, c0 + j, z);
      r[j] = __float_as_uint(z);
    }
    tmem_st32(taddr + (uint32_t)c0, r);
  }
  tmem_wait_st();
}

template <int H, typename IdxT>
__global__ void __launch_bounds__(THREADS, 1)
    linear_topk_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                       const float* __restrict__ bias, int64_t n_rows, int f_in, int k, float* __restrict__ sp_data,
                       IdxT* __restrict__ sp_idx, float* __restrict__ z_out, int64_t ld_z) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the dynamic shared memory base (SW128 atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kblocks = f_in / BK;
  uint8_t* sW = smem;                                        // kblocks x [H rows x 128 B]
  uint8_t* sX = sW + (size_t)kblocks * H * 128;              // STAGES x [BM rows x 128 B]
  float* bias_s = reinterpret_cast<float*>(sX + (size_t)STAGES * BM * 128);
  Barriers* bars = reinterpret_cast<Barriers*>((reinterpret_cast<uintptr_t>(bias_s + H) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (n_rows + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->tfull[a], 1);
      mbar_init(&bars->tempty[a], EPI_WARPS / 2);  // the 4 warps of the group that owns stage a
    }
    mbar_init(&bars->wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {  // TMEM: 2 accumulator stages x H fp32 columns (power of two >= 32)
    const uint32_t cols = 2 * H <= 32 ? 32 : (2 * H <= 64 ? 64 : (2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512)));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&bars->tmem_base)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = threadIdx.x; c < H; c += blockDim.x) bias_s[c] = bias ? bias[c] : 0.0f;
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      mbar_expect_tx(&bars->wbar, (uint32_t)(kblocks * H * 128));
      for (int kb = 0; kb < kblocks; ++kb) tma_load_2d(sW + (size_t)kb * H * 128, &map_w, &bars->wbar, kb * BK, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_parked(&bars->empty[stage], phase ^ 1u);
          mbar_expect_tx(&bars->full[stage], BM * 128);
          tma_load_2d(sX + (size_t)stage * BM * 128, &map_x, &bars->full[stage], kb * BK, (int)(t * BM));
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, H);
      mbar_wait(&bars->wbar, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int a = it & 1;
        mbar_wait_parked(&bars->tempty[a], ((it >> 1) & 1) ^ 1u);
        fence_after();
        const uint32_t d = tmem + (uint32_t)(a * H);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_parked(&bars->full[stage], phase);
          fence_after();
          const uint64_t adesc = desc_sw128(s32(sX + (size_t)stage * BM * 128));
          const uint64_t bdesc = desc_sw128(s32(sW + (size_t)kb * H * 128));
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)  // advance 16 bf16 = 32 bytes inside the swizzle atom
            umma_bf16(d, adesc + (uint64_t)(2 * kk), bdesc + (uint64_t)(2 * kk), idesc, (kb | kk) != 0 ? 1u : 0u);
          umma_commit(&bars->empty[stage]);  // frees the X slot when these MMAs complete
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        umma_commit(&bars->tfull[a]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ===== epilogue: thread-per-row exact top-k from TMEM =====
    const int q = warp & 3;                  // TMEM lane quarter this warp may access
    const int grp = (warp - 2) >> 2;         // group grp handles the CTA's tiles it = grp, grp + 2, ...
    float p_prev = NAN;
    const float zq = 1.41421356f * erfinvf(1.0f - 2.0f * (float)k / (float)H);  // Phi^-1(1 - k/H)
    int it = grp;
    for (int64_t t = blockIdx.x + (int64_t)grp * gridDim.x; t < n_tiles; t += 2 * (int64_t)gridDim.x, it += 2) {
      const int a = it & 1;
      mbar_wait(&bars->tfull[a], (it >> 1) & 1);
      fence_after();
      const int64_t row0 = t * BM + 32 * q;  // this warp's 32 rows
      const int64_t g = row0 + lane;
      const bool valid = g < n_rows;
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * H);

      // pass 0: range (+ optional z_out)
      float mn[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
      bias_pass<H>(taddr, bias_s, [&](int j, int c, float z) {
        mn[j & 3] = fminf(mn[j & 3], z);
        mx[j & 3] = fmaxf(mx[j & 3], z);
        s1[j & 3] += z;
        s2[j & 3] = fmaf(z, z, s2[j & 3]);
        if (z_out != nullptr && valid) z_out[g * ld_z + c] = z;
      });
      const float vmin = fminf(fminf(mn[0], mn[1]), fminf(mn[2], mn[3]));
      const float vmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      // phase 1: pivot probes (exact when exactly k values exceed the pivot).  tcgen05.ld is warp-collective, so
      // every pass is executed by the whole warp; a lane whose row is settled (or stalled) ignores the result.
      float lo = nextafterf(vmin, -INFINITY), hi = vmax, flo = (float)(H - k), fhi = -(float)k;
      // first probe: the row's Gaussian quantile estimate mean + std * Phi^-1(1 - k/H) (a heuristic start only;
      // the count decides), falling back to the previous row's pivot when the estimate is out of the bracket
      const float mean = ((s1[0] + s1[1]) + (s1[2] + s1[3])) * (1.0f / H);
      const float var = fmaxf(((s2[0] + s2[1]) + (s2[2] + s2[3])) * (1.0f / H) - mean * mean, 0.0f);
      const float sd = sqrtf(var);
      float p = fmaf(sd, zq, mean);
      if (!(p > lo && p < hi)) p = p_prev;
      // count slope at the quantile under the same Gaussian model, H * phi(zq) / sd: the second probe is a
      // Newton step from the first (the warp runs until its slowest row settles, so the tail matters)
      const float slope = (float)H * 0.39894228f * __expf(-0.5f * zq * zq) / sd;
      float piv = NAN;
      int side = 0;
      bool done = false, searching = true;
#pragma unroll 1
      for (int probe = 0; probe < 24; ++probe) {
        if (searching && !(p > lo && p < hi)) {
          p = lo + (hi - lo) * __fdividef(flo, flo - fhi);
          if (!(p > lo && p < hi)) p = 0.5f * lo + 0.5f * hi;
          if (!(p > lo && p < hi)) searching = false;  // fp32 stall: exact fallback below
        }
        if (!__any_sync(FULL, searching)) break;
        int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // independent partial counts (no serial add chain)
        const float pp = p;
        row_pass<H>(taddr, [&](int j, int, float z) { c8[j & 7] += z > pp ? 1 : 0; });
        const int cnt = ((c8[0] + c8[1]) + (c8[2] + c8[3])) + ((c8[4] + c8[5]) + (c8[6] + c8[7]));
        if (searching) {
          if (cnt == k) {
            piv = p;
            done = true;
            searching = false;
          } else {
            const float p0 = p;
            if (cnt > k) {
              lo = p; flo = (float)(cnt - k); if (side == 1) fhi *= 0.5f; side = 1;
            } else {
              hi = p; fhi = (float)(cnt - k); if (side == -1) flo *= 0.5f; side = -1;
            }
            p = NAN;
            if (probe == 0 && slope > 0.0f) {
              const float qn = p0 + (float)(cnt - k) / slope;
              if (qn > lo && qn < hi) p = qn;
            }
          }
        }
      }
      // phase 2 (exact fallback for rows phase 1 could not split): MSB-first descent to the k-th largest key T,
      // run by the whole warp when any lane needs it
      uint32_t T = 0u;
      int need = 0;
      if (__any_sync(FULL, !done)) {
#pragma unroll 1
        for (int bit = 31; bit >= 0; --bit) {
          const uint32_t cand = T | (1u << bit);
          int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          row_pass<H>(taddr, [&](int j, int, float z) { c8[j & 7] += f2key(z) >= cand ? 1 : 0; });
          const int cnt = ((c8[0] + c8[1]) + (c8[2] + c8[3])) + ((c8[4] + c8[5]) + (c8[6] + c8[7]));
          if (cnt >= k) T = cand;
        }
        int gt = 0;
        row_pass<H>(taddr, [&](int, int, float z) { gt += f2key(z) > T ? 1 : 0; });
        need = k - gt;
      }
      if (done) p_prev = piv;
      // emit in ascending column order into the padded staging row
      int pos = 0, eq = 0;
      row_pass<H>(taddr, [&](int, int c, float z) {
        bool s;
        if (done) {
          s = z > piv;
        } else {
          const uint32_t kz = f2key(z);
          s = kz > T || (kz == T && eq < need);
          eq += (kz == T) ? 1 : 0;
        }
        if (s && valid) {
          sp_data[g * k + pos] = z;
          sp_idx[g * k + pos] = (IdxT)c;
        }
        pos += s ? 1 : 0;
      });
      // the accumulator stage can be reused by the MMA warp
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->tempty[a]);
      __syncwarp();
    }
  }
  __syncthreads();
  if (warp == 2) {
    fence_after();
    const uint32_t cols = 2 * H <= 32 ? 32 : (2 * H <= 64 ? 64 : (2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512)));
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map: rows x cols (cols contiguous), box = box_rows x 64 cols, 128-byte swizzle
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int H, typename IdxT>
maxk_status_t run(const void* x, int64_t n, int f_in, int64_t ldx, const void* w_t, int64_t ldw, const float* bias,
                  int k, float* data, void* idx, float* z, int64_t ldz, cudaStream_t st) {
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, (uint64_t)n, (uint64_t)f_in, (uint64_t)ldx, BM) ||
      !make_map(&mw, w_t, (uint64_t)H, (uint64_t)f_in, (uint64_t)ldw, H))
    return fail(MAXK_ERR_CUDA, "linear_topk: cuTensorMapEncodeTiled failed (alignment or driver)");
  const size_t smem = 1024 /*align slack*/ + (size_t)(f_in / BK) * H * 128 + (size_t)STAGES * BM * 128 + H * 4 +
                      16 + sizeof(Barriers);
  if (smem > 227 * 1024) return fail(MAXK_ERR_UNSUPPORTED, "linear_topk: %zu B of shared memory needed", smem);
  auto kern = linear_topk_kernel<H, IdxT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(MAXK_ERR_CUDA, "linear_topk: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const int64_t tiles = (n + BM - 1) / BM;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  kern<<<grid, THREADS, smem, st>>>(mx, mw, bias, n, f_in, k, data, static_cast<IdxT*>(idx), z, ldz);
  note_launch();
  return check_launch("linear_topk_kernel");
}

}  // namespace

maxk_status_t launch_linear_topk(const void* x, int64_t n, int f_in, int64_t ldx, const void* w_t, int64_t ldw,
                                 const float* bias, int h, int k, int idx_bytes, float* data, void* idx, float* z,
                                 int64_t ldz, cudaStream_t st) {
  if (h == 256)
    return idx_bytes == 1 ? run<256, uint8_t>(x, n, f_in, ldx, w_t, ldw, bias, k, data, idx, z, ldz, st)
                          : run<256, uint16_t>(x, n, f_in, ldx, w_t, ldw, bias, k, data, idx, z, ldz, st);
  if (h == 128)
    return idx_bytes == 1 ? run<128, uint8_t>(x, n, f_in, ldx, w_t, ldw, bias, k, data, idx, z, ldz, st)
                          : run<128, uint16_t>(x, n, f_in, ldx, w_t, ldw, bias, k, data, idx, z, ldz, st);
  return fail(MAXK_ERR_UNSUPPORTED, "linear_topk supports h in {128, 256} (h=%d)", h);
}

}  // namespace maxk
