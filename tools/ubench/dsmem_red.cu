// Microbenchmark: random-column float accumulation into per-warp 256-float row buffers.
//   mode 0: local shared-memory read-modify-write (LDS + FADD + STS), the forward kernel's accumulation
//   mode 1: red.shared::cluster.add.f32 into the PEER CTA's buffer (cluster of 2; native ATOM.ADD.F32)
//   mode 2: red.shared::cluster.add.f32 into the OWN CTA's buffer (compiles to a CAS loop)
//   mode 3: local RMW into one of 2 bank-shifted replicas (shift 16), lanes alternating replicas within a
//           __match_any_sync group of equal banks (the forward's conflict-spreading candidate)
// Each warp issues ITERS instructions of 32 random columns (k=32 entries of one edge per instruction).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256) kern(float* out, int iters, unsigned seed) {
  __shared__ float buf[8][MODE == 3 ? 512 : 256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = lane; c < (MODE == 3 ? 512 : 256); c += 32) buf[w][c] = 0.f;
  asm volatile("barrier.cluster.arrive; barrier.cluster.wait;" ::: "memory");
  unsigned rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const unsigned base = (unsigned)__cvta_generic_to_shared(&buf[w][0]);
  unsigned peer = base;
  if (MODE == 1) asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(base), "r"(rank ^ 1u));
  if (MODE == 2) asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(base), "r"(rank));
  unsigned x = seed ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const unsigned col = x >> 24;  // 0..255
    const float v = 1.0f;
    if (MODE == 3) {
      const unsigned bank = col & 31u;
      const unsigned grp = __match_any_sync(0xffffffffu, bank);
      const unsigned rep = __popc(grp & ((1u << lane) - 1u)) & 1u;
      const unsigned a = base + 4u * (rep * 256u + (col & ~31u) + ((bank + rep * 16u) & 31u));
      float o;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(a));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(o + v));
      __syncwarp();
    } else if (MODE == 0) {
      float o;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(base + 4u * col));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + 4u * col), "f"(o + v));
      __syncwarp();
    } else {
      asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(peer + 4u * col), "f"(v) : "memory");
    }
  }
  asm volatile("barrier.cluster.arrive; barrier.cluster.wait;" ::: "memory");
  float s = 0.f;
  for (int c = lane; c < 256; c += 32) s += buf[w][c];
  if (s == -1.f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 20000;
  for (int mode : {0, 3, 1}) {
    for (int cps = 2; cps <= (mode == 1 ? 2 : 6); cps += 2) {  // CTAs per SM
      const int blocks = sms * cps;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) kern<0><<<blocks, 256>>>(out, iters, 1u);
        if (mode == 1) kern<1><<<blocks, 256>>>(out, iters, 1u);
        if (mode == 2) kern<2><<<blocks, 256>>>(out, iters, 1u);
        if (mode == 3) kern<3><<<blocks, 256>>>(out, iters, 1u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      const double instr = (double)blocks * 8 * iters;  // warp-instructions of 32 entries
      printf("mode %d ctas/SM %d: %.3f ms, %.2f SM-cycles(1.965GHz) per 32-entry warp op per SM %s\n", mode, cps, ms,
             ms * 1e-3 * 1.965e9 * sms / instr, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
