// scatter.cu — MaxK backward scatter (§3.1 Def. ii):
//   dx[r, sp_idx[r,t]] = d_sp_data[r,t], zero elsewhere.
// One warp per row: zero an h-float shared-memory row, scatter the k values (distinct columns: no race),
// then write the dense row with coalesced float4 stores.  HBM-bound (4h bytes written per row).
#include <algorithm>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

constexpr int SC_THREADS = 256;

template <typename IdxT, bool VEC>
__global__ void __launch_bounds__(SC_THREADS) cbsr_scatter_kernel(const float* __restrict__ g,
                                                                  const IdxT* __restrict__ idx, int64_t n, int h,
                                                                  int k, float* __restrict__ dx, int64_t ld) {
  extern __shared__ float4 smem4[];
  float* buf = reinterpret_cast<float*>(smem4) + (threadIdx.x >> 5) * h;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  for (int64_t r = warp; r < n; r += nwarps) {
    if (VEC) {
      for (int c = lane * 4; c < h; c += 128) *reinterpret_cast<float4*>(buf + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int c = lane; c < h; c += 32) buf[c] = 0.0f;
    }
    __syncwarp();
    for (int t = lane; t < k; t += 32) buf[ld_keep_idx(idx + r * k + t, pol)] = ld_stream_f32(g + r * k + t, pol);
    __syncwarp();
    float* dst = dx + r * ld;
    if (VEC) {
      for (int c = lane * 4; c < h; c += 128) *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<float4*>(buf + c);
    } else {
      for (int c = lane; c < h; c += 32) dst[c] = buf[c];
    }
    __syncwarp();
  }
}

template <typename IdxT>
maxk_status_t run(const float* g, const void* idx, int64_t n, int h, int k, float* dx, int64_t ld, cudaStream_t st) {
  const bool vec = (h % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(dx) & 15u) == 0);
  const int warps = (int)std::min<int64_t>(SC_THREADS / 32, (227 * 1024) / ((int64_t)h * 4));
  const size_t smem = (size_t)warps * h * sizeof(float);
  auto kern = vec ? cbsr_scatter_kernel<IdxT, true> : cbsr_scatter_kernel<IdxT, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(MAXK_ERR_CUDA, "cbsr_scatter: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
  }
  int64_t blocks = (n + warps - 1) / warps;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, warps * 32, smem, st>>>(g, static_cast<const IdxT*>(idx), n, h, k, dx, ld);
  note_launch();
  return check_launch("cbsr_scatter_kernel");
}

}  // namespace

maxk_status_t launch_cbsr_scatter(const float* g, const void* idx, int64_t n, int h, int k, int idx_bytes, float* dx,
                                  int64_t ld, cudaStream_t st) {
  return idx_bytes == 1 ? run<uint8_t>(g, idx, n, h, k, dx, ld, st) : run<uint16_t>(g, idx, n, h, k, dx, ld, st);
}

}  // namespace maxk
