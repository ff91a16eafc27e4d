// ubench.cu — microbenchmarks of the ceilings that bound the aggregation kernels.
// Measurement tooling only (not the product): each kernel isolates one component of the k=32 inner loop
// of spgemm_fwd_vec_kernel / sspmm_bwd_vec_kernel with the same lane mapping (8 lanes x 4 entries per edge,
// 4 edges per warp step, 4 steps in flight):
//   ub_smem_rmw     shared-memory read-modify-write of 4 columns per lane into a per-sub-warp 256-float row
//                   buffer; the column sets are real CBSR index rows staged in shared memory (no global loads)
//   ub_lds_gather   the backward's read-only gather of 4 columns per lane from one staged 256-float row
//   ub_cbsr_gather  the forward's global part only: stream col_idx/val, gather the CBSR row of every edge
//                   (LDG.128 sp_data + LDG.32 sp_idx), fold into registers (no shared memory)
//   ub_red          the backward's reduction part only: one red.global.add.v4.f32 per lane per edge into
//                   d_sp_data[col, :] (no index load, no shared memory)
// All kernels are grid-stride over a flat edge range; results are folded into `sink` to defeat DCE.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr unsigned FULL = 0xffffffffu;

__global__ void __launch_bounds__(256) ub_smem_rmw(const uint8_t* __restrict__ idx_rows, int n_idx_rows,
                                                   int64_t n_edges, float* sink) {
  __shared__ float buf[8][4][256];
  __shared__ uint32_t tab[512][8];  // 512 CBSR index rows of 32 bytes
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sub = lane >> 3, p = lane & 7;
  for (int i = threadIdx.x; i < 512 * 8; i += blockDim.x)
    tab[i >> 3][i & 7] = reinterpret_cast<const uint32_t*>(idx_rows)[(i >> 3) % n_idx_rows * 8 + (i & 7)];
  for (int i = lane; i < 4 * 256; i += 32) (&buf[w][0][0])[i] = 0.f;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(&buf[w][sub][0]);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float wgt = 0.5f;
  // each warp step = 4 edges (one per sub-warp); 4 steps per iteration
  for (int64_t e = warp * 16; e < n_edges; e += nw * 16) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t x = tab[(uint32_t)(e + s * 4 + sub) & 511][p];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint32_t a = base + 4u * ((x >> (8 * v)) & 0xffu);
        float o;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(a));
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(fmaf(wgt, 1.0f, o)));
      }
      __syncwarp();
    }
  }
  __syncwarp();
  if (lane == 0) atomicAdd(sink, buf[w][0][0]);
}

__global__ void __launch_bounds__(256) ub_lds_gather(const uint8_t* __restrict__ idx_rows, int n_idx_rows,
                                                     int64_t n_edges, float* sink) {
  __shared__ float buf[8][256];
  __shared__ uint32_t tab[512][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sub = lane >> 3, p = lane & 7;
  for (int i = threadIdx.x; i < 512 * 8; i += blockDim.x)
    tab[i >> 3][i & 7] = reinterpret_cast<const uint32_t*>(idx_rows)[(i >> 3) % n_idx_rows * 8 + (i & 7)];
  for (int i = lane; i < 256; i += 32) buf[w][i] = (float)i;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(&buf[w][0]);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t e = warp * 16; e < n_edges; e += nw * 16) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t x = tab[(uint32_t)(e + s * 4 + sub) & 511][p];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float o;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(base + 4u * ((x >> (8 * v)) & 0xffu)));
        acc += o;
      }
    }
  }
  if (acc == -1.f) *sink = acc;
}

__global__ void __launch_bounds__(256) ub_cbsr_gather(const int32_t* __restrict__ col, const float* __restrict__ val,
                                                      int64_t n_edges, const float* __restrict__ sp_data,
                                                      const uint8_t* __restrict__ sp_idx, float* sink) {
  const int lane = threadIdx.x & 31, sub = lane >> 3, p = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  uint32_t xacc = 0u;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    int cj = 0;
    float cv = 0.f;
    if (lane < nb) {
      cj = __ldg(col + eb + lane);
      cv = __ldg(val + eb + lane);
    }
    for (int q = 0; q + 16 <= nb; q += 16) {
      float4 d[4];
      uint32_t x[4];
      float wv[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int j = __shfl_sync(FULL, cj, q + s * 4 + sub);
        wv[s] = __shfl_sync(FULL, cv, q + s * 4 + sub);
        d[s] = __ldg(reinterpret_cast<const float4*>(sp_data + (int64_t)j * 32) + p);
        x[s] = __ldg(reinterpret_cast<const uint32_t*>(sp_idx + (int64_t)j * 32) + p);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        acc = fmaf(wv[s], d[s].x + d[s].y + d[s].z + d[s].w, acc);
        xacc ^= x[s];
      }
    }
  }
  if (acc == -1.f && xacc == 7u) *sink = acc;
}

__global__ void __launch_bounds__(256) ub_red(const int32_t* __restrict__ col, int64_t n_edges, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, sub = lane >> 3, p = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    const int cj = lane < nb ? __ldg(col + eb + lane) : 0;
    for (int q = 0; q + 16 <= nb; q += 16) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int j = __shfl_sync(FULL, cj, q + s * 4 + sub);
        float* a = out + (int64_t)j * 32 + p * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
      }
    }
  }
}

// scalar variant: 32 lanes x 4 B per edge, one edge per instruction
__global__ void __launch_bounds__(256) ub_red_scalar(const int32_t* __restrict__ col, int64_t n_edges,
                                                     float* __restrict__ out, int mask_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    const int cj = lane < nb ? __ldg(col + eb + lane) : 0;
    for (int q = 0; q < nb; ++q) {
      const int j = __shfl_sync(FULL, cj, q) & mask_rows;
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(out + (int64_t)j * 32 + lane), "f"(1.f) : "memory");
    }
  }
}

// v4 variant with the destination rows folded into a small target (j & mask_rows): contention / size test
__global__ void __launch_bounds__(256) ub_red_masked(const int32_t* __restrict__ col, int64_t n_edges,
                                                     float* __restrict__ out, int mask_rows) {
  const int lane = threadIdx.x & 31, sub = lane >> 3, p = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    const int cj = lane < nb ? __ldg(col + eb + lane) : 0;
    for (int q = 0; q + 16 <= nb; q += 16) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int j = __shfl_sync(FULL, cj, q + s * 4 + sub) & mask_rows;
        float* a = out + (int64_t)j * 32 + p * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
      }
    }
  }
}

// plain 128-B stores of the same pattern (write-path bandwidth, no atomics): distinguishes the L2 atomic ALUs
// from the SM -> L2 write path as the reduction ceiling
__global__ void __launch_bounds__(256) ub_stg(const int32_t* __restrict__ col, int64_t n_edges, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, sub = lane >> 3, p = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    const int cj = lane < nb ? __ldg(col + eb + lane) : 0;
    for (int q = 0; q + 16 <= nb; q += 16) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int j = __shfl_sync(FULL, cj, q + s * 4 + sub);
        *reinterpret_cast<float4*>(out + (int64_t)j * 32 + p * 4) = make_float4(1.f, 1.f, 1.f, (float)q);
      }
    }
  }
}

// TMA bulk reduction: the sub-warp writes its edge's 128 B into a shared slot, one lane issues
// cp.reduce.async.bulk .add.f32 of 128 B to d_sp_data[j, :].  Ring of 4 slots per sub-warp.
__global__ void __launch_bounds__(256) ub_red_bulk(const int32_t* __restrict__ col, int64_t n_edges,
                                                   float* __restrict__ out) {
  __shared__ __align__(128) float slots[8][4][4][32];  // [warp][sub][ring][32 floats]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sub = lane >> 3, p = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int ring = 0;
  for (int64_t eb = warp * 32; eb < n_edges; eb += nw * 32) {
    const int nb = (int)min((int64_t)32, n_edges - eb);
    const int cj = lane < nb ? __ldg(col + eb + lane) : 0;
    for (int q = 0; q + 4 <= nb; q += 4) {
      const int j = __shfl_sync(FULL, cj, q + sub);
      float* slot = &slots[w][sub][ring][0];
      if (p == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");  // slot reuse after 4 groups
      __syncwarp();
      *reinterpret_cast<float4*>(slot + p * 4) = make_float4(1.f, 1.f, 1.f, 1.f);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (p == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(slot);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;" ::"l"(
                         out + (int64_t)j * 32), "r"(sa) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ring = (ring + 1) & 3;
    }
  }
  if (p == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename K, typename... A>
float time_it(K kern, int reps, A... args) {
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  kern<<<blocks, 256>>>(args...);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) kern<<<blocks, 256>>>(args...);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? ms / reps : -1.f;
}

}  // namespace

extern "C" {
// Each returns the mean milliseconds per launch over `reps` launches (-1 on a CUDA error).
float ubench_smem_rmw(const uint8_t* idx_rows, int n_idx_rows, int64_t n_edges, float* sink, int reps) {
  return time_it(ub_smem_rmw, reps, idx_rows, n_idx_rows, n_edges, sink);
}
float ubench_lds_gather(const uint8_t* idx_rows, int n_idx_rows, int64_t n_edges, float* sink, int reps) {
  return time_it(ub_lds_gather, reps, idx_rows, n_idx_rows, n_edges, sink);
}
float ubench_cbsr_gather(const int32_t* col, const float* val, int64_t n_edges, const float* sp_data,
                         const uint8_t* sp_idx, float* sink, int reps) {
  return time_it(ub_cbsr_gather, reps, col, val, n_edges, sp_data, sp_idx, sink);
}
float ubench_red(const int32_t* col, int64_t n_edges, float* out, int reps) {
  return time_it(ub_red, reps, col, n_edges, out);
}
float ubench_red_scalar(const int32_t* col, int64_t n_edges, float* out, int mask_rows, int reps) {
  return time_it(ub_red_scalar, reps, col, n_edges, out, mask_rows);
}
float ubench_red_masked(const int32_t* col, int64_t n_edges, float* out, int mask_rows, int reps) {
  return time_it(ub_red_masked, reps, col, n_edges, out, mask_rows);
}
float ubench_stg(const int32_t* col, int64_t n_edges, float* out, int reps) {
  return time_it(ub_stg, reps, col, n_edges, out);
}
float ubench_red_bulk(const int32_t* col, int64_t n_edges, float* out, int reps) {
  return time_it(ub_red_bulk, reps, col, n_edges, out);
}
}
