// linear_topk.cu — Eq. 1 fused: h(X) = max-k (X·W + b) -> CBSR.
//
// One persistent CTA per SM, warp-specialised (sm_100a tcgen05 / TMEM / TMA):
//   warp 0      TMA producer: loads W^T once (resident in shared memory, 128B-swizzled K-major), then streams
//               128 x 64 bf16 tiles of X through a STAGES-deep mbarrier ring;
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32,
//               M=128, N=h, K=16) into a double-buffered TMEM accumulator (2 x h columns);
//   warps 2..9  epilogue, all eight on every tile: the tile's z = acc + b is staged through shared memory in two
//               64-row halves (the two warps of each TMEM lane quarter copy it with tcgen05.ld.32x32b.x32, 16-byte
//               units XOR-swizzled by row so both the row-major writes and the row reads are conflict-free), then
//               each warp selects 8 rows of the half warp-per-row with the standalone kernel's selection
//               (topk_row.cuh: seeded warm start, extraction finish, exact key-descent fallback) and writes them
//               with coalesced stores.  The TMEM stage is released as soon as the second half is staged, so the
//               tensor cores fill it with tile t+2 while tile t is selected.
// The selection is the exact top-k of the fp32 z the kernel computes (ties -> lower column, -0 == +0),
// identical to maxk_topk_cbsr applied to z; z itself can be written out (z_out) for verification.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>

#include "maxk_internal.cuh"
#include "topk_row.cuh"

namespace maxk {
namespace {

constexpr int BM = 128;          // rows per tile (UMMA M)
constexpr int BK = 64;           // bf16 elements per 128-byte swizzle row (one k-block)
constexpr int STAGES = 2;        // X tile ring depth (shared memory: W^T + X ring + the 64-row z stage)
#ifndef MAXK_F4_EPI_WARPS
#define MAXK_F4_EPI_WARPS 24  // measured: 8 -> 0.255 ms, 16 -> 0.161, 24 -> 0.153, 28 -> 0.159 (Reddit-shaped rows)
#endif
constexpr int EPI_WARPS = MAXK_F4_EPI_WARPS;  // EPI_WARPS / 4 per TMEM lane quarter for staging; all of them select
static_assert(EPI_WARPS % 4 == 0 && EPI_WARPS <= 30, "epilogue warps: a multiple of 4, at most 30 (1024 threads)");
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
__device__ __forceinline__ void named_sync_epi() {  // the eight epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
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
  float* sZ = reinterpret_cast<float*>(sX + (size_t)STAGES * BM * 128);  // 64 rows x H fp32, 16-B units swizzled
  float* bias_s = sZ + 64 * H;
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
      mbar_init(&bars->tempty[a], 1);  // one arrival once the tile's second half is staged
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
    // ===== epilogue: z staged through shared memory, then warp-per-row selection =====
    constexpr int E = H / 32;                // values per lane of a row (float4 groups of the standalone kernel)
    constexpr int NG = E / 4;
    const int e = warp - 2;                  // epilogue warp 0 .. EPI_WARPS - 1
    const int q = warp & 3;                  // the TMEM lane quarter this warp may access
    constexpr int STAGERS = EPI_WARPS < 16 ? EPI_WARPS : 16;  // warps that copy TMEM to the stage
    constexpr int CPARTS = STAGERS / 4;      // stagers per TMEM lane quarter: each copies H / CPARTS columns
    const int cpart = e >> 2;                // which part of the columns it stages
    const uint32_t zbase = s32(sZ);
    // row r (0..63 of the half), 16-byte unit u of z at zbase + 4 (r H + 4 (u ^ (r & 7))): XOR-swizzled so a
    // quarter-warp of row-major STS.128 (8 rows, one unit) and a warp's LDS.128 of one row both hit 32 banks
    auto zaddr = [&](int r, int u) { return zbase + 4u * (uint32_t)(r * H + 4 * (u ^ (r & 7))); };
    uint32_t col[E];
#pragma unroll
    for (int i = 0; i < E; ++i) col[i] = (uint32_t)((i / 4) * 128 + lane * 4 + (i % 4));
    PivotState ps = pivot_state(k, H);
    int it = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int a = it & 1;
      mbar_wait(&bars->tfull[a], (it >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        if (e < STAGERS && (q >> 1) == hf) {  // stage TMEM lanes 32 q .. 32 q + 31 (rows 64 hf + 32 (q & 1) + lane), one column part
          const int r = 32 * (q & 1) + lane;
          const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * H);
#pragma unroll 1
          for (int c0 = cpart * (H / CPARTS); c0 < (cpart + 1) * (H / CPARTS); c0 += 32) {
            uint32_t v32[32];
            tmem_ld32(taddr + (uint32_t)c0, v32);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              sts128(zaddr(r, (c0 + j) >> 2), __uint_as_float(v32[j]) + bias_s[c0 + j],
                     __uint_as_float(v32[j + 1]) + bias_s[c0 + j + 1], __uint_as_float(v32[j + 2]) + bias_s[c0 + j + 2],
                     __uint_as_float(v32[j + 3]) + bias_s[c0 + j + 3]);
          }
        }
        fence_before();
        named_sync_epi();  // the half is staged (and, after the second, every TMEM read of this tile is done)
        if (hf == 1 && e == 0 && lane == 0) mbar_arrive(&bars->tempty[a]);
        // warp e selects rows e, e + EPI_WARPS, ... of the half; a row's slot is its own staging area afterwards
#pragma unroll 1
        for (int r = e; r < 64; r += EPI_WARPS) {
          const int64_t g = t * BM + 64 * hf + r;
          if (g >= n_rows) break;
          float v[E];
#pragma unroll
          for (int gg = 0; gg < NG; ++gg) {
            const float4 f = lds128f(zaddr(r, 32 * gg + lane));
            v[4 * gg] = f.x; v[4 * gg + 1] = f.y; v[4 * gg + 2] = f.z; v[4 * gg + 3] = f.w;
            if (z_out != nullptr)
              *reinterpret_cast<float4*>(z_out + g * ld_z + 128 * gg + 4 * lane) = f;
          }
          __syncwarp();
          const uint32_t slot = zbase + 4u * (uint32_t)(r * H);  // values at +0, columns at +256 bytes (k <= 64)
          select_row<E, false, 256>(v, col, k, ps, slot, lane);
          __syncwarp();
          for (int t0 = 0; t0 < k; t0 += 32) {
            const int tt = t0 + lane;
            if (tt < k) {
              sp_data[g * k + tt] = sZ[r * H + tt];
              sp_idx[g * k + tt] = (IdxT)__float_as_uint(sZ[r * H + 64 + tt]);
            }
          }
          __syncwarp();
        }
        named_sync_epi();  // the half's rows are done before the next half is staged over them
      }
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
  const size_t smem = 1024 /*align slack*/ + (size_t)(f_in / BK) * H * 128 + (size_t)STAGES * BM * 128 +
                      (size_t)64 * H * 4 /*z stage*/ + H * 4 + 16 + sizeof(Barriers);
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
