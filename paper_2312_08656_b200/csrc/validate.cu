// validate.cu — debug-only checks of the input-VALUE contract of include/maxk.h (never on the hot path):
// the layer calls trust row_ptr monotonicity, col_idx < n_cols and strictly ascending sp_idx < h (SPEC.md:26-27,
// SPEC.md:110 and 169; SURVEY §8(b) "maxk_validate_csr / maxk_validate_cbsr ... outside the hot path").
#include <functional>

#include "maxk_internal.cuh"

namespace maxk {
namespace {

// counts[0]: rows with row_ptr[i+1] < row_ptr[i]; counts[1]: edges with col_idx outside [0, n_cols)
__global__ void validate_csr_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                    int64_t n_rows, int64_t n_cols, unsigned long long* counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long bad_rows = 0, bad_cols = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += stride) {
    const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
    if (e1 < e0) { ++bad_rows; continue; }
    for (int64_t e = e0; e < e1; ++e) bad_cols += (col[e] < 0 || (int64_t)col[e] >= n_cols) ? 1ull : 0ull;
  }
  if (bad_rows) atomicAdd(counts + 0, bad_rows);
  if (bad_cols) atomicAdd(counts + 1, bad_cols);
}

// counts[0]: CBSR rows whose indices are not strictly ascending or not < h
template <typename IdxT>
__global__ void validate_cbsr_kernel(const IdxT* __restrict__ idx, int64_t n_rows, int k, int h,
                                     unsigned long long* counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long bad = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += stride) {
    const IdxT* row = idx + r * (int64_t)k;
    bool ok = (int)row[k - 1] < h;
    for (int t = 1; t < k && ok; ++t) ok = row[t - 1] < row[t];
    bad += ok ? 0ull : 1ull;
  }
  if (bad) atomicAdd(counts, bad);
}

maxk_status_t run_counts(unsigned long long* host, int n, cudaStream_t st,
                         const std::function<void(unsigned long long*)>& launch) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, n * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(d, 0, n * sizeof(unsigned long long), st);
  if (e == cudaSuccess) {
    launch(d);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d) cudaFree(d);
  if (e != cudaSuccess) return fail(MAXK_ERR_CUDA, "validate: %s", cudaGetErrorString(e));
  return MAXK_OK;
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace
}  // namespace maxk

using namespace maxk;

extern "C" {

maxk_status_t maxk_validate_csr(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols,
                                maxk_stream_t stream, int64_t* bad_rows, int64_t* bad_cols) {
  if (n_rows < 0 || n_cols < 0) return fail(MAXK_ERR_INVALID_ARGUMENT, "negative n_rows or n_cols");
  if (n_rows > 0 && (!row_ptr || !col_idx)) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL row_ptr or col_idx");
  unsigned long long c[2] = {0, 0};
  if (n_rows > 0) {
    cudaStream_t st = (cudaStream_t)stream;
    maxk_status_t s = run_counts(c, 2, st, [&](unsigned long long* d) {
      validate_csr_kernel<<<grid_for(n_rows), 256, 0, st>>>(row_ptr, col_idx, n_rows, n_cols, d);
    });
    if (s != MAXK_OK) return s;
  }
  if (bad_rows) *bad_rows = (int64_t)c[0];
  if (bad_cols) *bad_cols = (int64_t)c[1];
  return MAXK_OK;
}

maxk_status_t maxk_validate_cbsr(const void* sp_idx, int64_t n_rows, int32_t h, int32_t k, int32_t idx_bytes,
                                 maxk_stream_t stream, int64_t* bad_rows) {
  if (n_rows < 0 || k < 1 || k > h || (idx_bytes != 1 && idx_bytes != 2))
    return fail(MAXK_ERR_INVALID_ARGUMENT, "bad n_rows, k=%d, h=%d or idx_bytes=%d", k, h, idx_bytes);
  if (n_rows > 0 && !sp_idx) return fail(MAXK_ERR_INVALID_ARGUMENT, "NULL sp_idx");
  unsigned long long c = 0;
  if (n_rows > 0) {
    cudaStream_t st = (cudaStream_t)stream;
    maxk_status_t s = run_counts(&c, 1, st, [&](unsigned long long* d) {
      if (idx_bytes == 1)
        validate_cbsr_kernel<uint8_t><<<grid_for(n_rows), 256, 0, st>>>((const uint8_t*)sp_idx, n_rows, k, h, d);
      else
        validate_cbsr_kernel<uint16_t><<<grid_for(n_rows), 256, 0, st>>>((const uint16_t*)sp_idx, n_rows, k, h, d);
    });
    if (s != MAXK_OK) return s;
  }
  if (bad_rows) *bad_rows = (int64_t)c;
  return MAXK_OK;
}

}  // extern "C"
