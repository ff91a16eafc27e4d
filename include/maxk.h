/*
 * maxk.h — C-ABI of the B200-native MaxK-GNN layer hot path (arXiv 2312.08656).
 *
 * Three operations, one per step of the paper's layer dataflow (Fig. 5):
 *   maxk_topk_cbsr   MaxK nonlinearity -> CBSR          Eq. 1 (§3.1); CBSR PAPER.md:326
 *   maxk_spgemm_fwd  Y = A · CBSR(X), row-wise product   Eq. 3 left; Alg. 1
 *   maxk_sspmm_bwd   dXs = (A^T · dY) at the CBSR mask   Eq. 3 right / Eq. 4; Alg. 2
 *                    (PAPER.md:447-468), reading R8 of DESIGN.md for its garbled line 9
 * plus the once-per-graph work plan (the paper's O(n) warp-partition meta-data), and B200
 * companions of these calls: the CBSR pair layout and the bank-balanced copies the forward reads
 * (maxk_topk_cbsr_pairs / _pairs_banked / _banked, maxk_spgemm_fwd_pairs, maxk_spgemm_fwd_replicated), the
 * accumulating forms and the exchanges fused into the kernels for the row-partitioned multi-GPU pass
 * (maxk_spgemm_fwd_acc, maxk_sspmm_bwd_acc, maxk_topk_cbsr_multi, maxk_sspmm_bwd_owners), the MaxK backward
 * scatter, Eq. 1 fused on the tensor cores, and debug validators / statistics.
 *
 * Conventions (all functions):
 *   - Every array argument is a DEVICE pointer (cudaMalloc'd or managed), unless stated otherwise.
 *   - The caller owns every array. The library owns only maxk_plan_t objects.
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream) and never
 *     synchronise, except maxk_plan_create, which synchronises `stream` once.
 *   - Nothing is allocated on the per-layer path; maxk_plan_create allocates the plan.
 *   - Outputs must not alias inputs.
 *   - Validation is host-side and happens before any launch; on error nothing is launched and the
 *     status says why (maxk_last_error_detail() gives a thread-local message).
 *   - Input VALUES are the caller's contract and are not checked on the hot path: row_ptr monotone,
 *     0 <= col_idx < n_cols, sp_idx entries < h and strictly ascending per row (the aggregation calls need them
 *     only distinct: they also take the bank-balanced order of maxk_topk_cbsr_banked), X finite (NaN input to
 *     top-k gives an unspecified selection; +-Inf are ordinary values).
 *   - Asynchronous device faults surface at the caller's next synchronisation with the stream.
 *
 * Layouts:
 *   X, Y, dY   fp32, row-major, n_rows x h with row stride ld (elements), ld >= h.
 *   CBSR       two separate blocks (the paper's adjacent sp_data / sp_index blocks):
 *              sp_data fp32 [n x k] row stride k, sp_idx uint8 (idx_bytes=1, h <= 256) or uint16
 *              (idx_bytes=2, h <= 65536) [n x k] row stride k, indices strictly ascending per row.
 *   CSR        row_ptr int64 [n_rows+1], col_idx int32 [nnz], val fp32 [nnz]. row_ptr[0] may be
 *              nonzero (a zero-copy row block); col_idx/val are then indexed absolutely.
 *              nnz must equal row_ptr[n_rows] - row_ptr[0].  Duplicate (i,j) entries are summed.
 *              The backward pass reads the SAME arrays as the CSC of A^T.
 *   n_cols may differ from n_rows: it is the number of CBSR rows the forward gathers from and the
 *   backward scatters to (the multi-GPU slot space).
 */
#ifndef MAXK_H_
#define MAXK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MAXK_OK = 0,
  MAXK_ERR_INVALID_ARGUMENT = 1, /* a size, stride, width or pointer argument is invalid */
  MAXK_ERR_UNSUPPORTED = 2,      /* valid but outside what this build implements (e.g. h too large) */
  MAXK_ERR_CUDA = 3,             /* a CUDA runtime call or launch failed (detail has the CUDA string) */
  MAXK_ERR_OUT_OF_MEMORY = 4     /* plan allocation failed */
} maxk_status_t;

typedef struct CUstream_st* maxk_stream_t; /* == cudaStream_t */
typedef struct maxk_plan maxk_plan_t;      /* opaque, library-owned */

/*
 * MaxK top-k -> CBSR (Eq. 1; "node-wise ... maximum k").
 * For each row r of x: select the k columns with the largest values, ranking by (value descending,
 * column ascending) under IEEE comparison (so -0.0 == +0.0 and the lower column wins the tie).
 * Writes sp_idx[r, 0..k) = the selected columns in ascending order, sp_data[r, t] = x[r, sp_idx[r, t]]
 * as an exact bit copy.
 *   x         [n_rows x h], row stride ld_x >= h            (read)
 *   k         1 <= k <= h
 *   idx_bytes 1 (requires h <= 256) or 2 (requires h <= 65536)
 *   sp_data   [n_rows x k] fp32                              (written)
 *   sp_idx    [n_rows x k] uint8/uint16                      (written)
 * Errors: INVALID_ARGUMENT for k < 1, k > h, bad idx_bytes, ld_x < h, NULL pointer with n_rows > 0;
 *         UNSUPPORTED for h > 1024 (register-resident row limit of this build).
 * n_rows == 0 is a no-op returning MAXK_OK.
 */
maxk_status_t maxk_topk_cbsr(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                             int32_t idx_bytes, float* sp_data, void* sp_idx, maxk_stream_t stream);

/*
 * Pair layout of the CBSR (a B200 companion of the two-block layout for k in {8, 16}):
 *   sp_pairs [n x k] of {uint32 value bits, uint32 column}, 8 bytes per entry, row stride 8k bytes (64 / 128),
 *   16-byte aligned base, entries in the same ascending column order as sp_idx, value bits identical to sp_data.
 * A k <= 16 row then lies in ONE 128-byte line and one load instruction brings an edge's values and indices,
 * where the two blocks cost two lines (two L1tex wavefronts) per gathered row in the forward pass.
 *
 * maxk_topk_cbsr_pairs: maxk_topk_cbsr (same selection, same sp_data / sp_idx) that also writes sp_pairs.
 *   Errors: as maxk_topk_cbsr; INVALID_ARGUMENT for a NULL or misaligned sp_pairs; UNSUPPORTED unless
 *   k in {8, 16} and h in {128, 256, 384, 512} with 16-byte aligned rows of x.
 */
maxk_status_t maxk_topk_cbsr_pairs(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                   int32_t idx_bytes, float* sp_data, void* sp_idx, void* sp_pairs,
                                   maxk_stream_t stream);

/*
 * maxk_topk_cbsr_pairs_banked (k = 16 only): maxk_topk_cbsr_pairs with the pairs in the mod-4-balanced order the
 * forward's NC = 8 row buffers read (lanes p = pi + 2m of entry group e share an accumulator copy whose bank is
 * 8 (c mod 4) + ...): class m = c mod 4, in ascending column order, takes position 2 (pi + 2m) + e of
 * the sets j = (e, pi) = (j / 2, j % 2) for j = 0, 1, 2, 3; the entries of a class beyond its fourth, in ascending
 * column order, fill the positions deficient classes leave free, ordered set 3 first, then by class.  sp_data /
 * sp_idx stay in column order.
 *   Errors: as maxk_topk_cbsr_pairs; UNSUPPORTED unless k = 16.
 */
maxk_status_t maxk_topk_cbsr_pairs_banked(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                          int32_t idx_bytes, float* sp_data, void* sp_idx, void* sp_pairs,
                                          maxk_stream_t stream);

/*
 * Bank-balanced entry order of the CBSR (a B200 companion of the column-ordered CBSR for the forward's replicated
 * row buffers, like the pair layout).  The paper fixes a CBSR row as k (value, column) entries
 * (Fig. 4); the SpGEMM and the SSpMM need the columns of a row distinct, not ascending.
 * maxk_topk_cbsr_banked: maxk_topk_cbsr (same selection, same sp_data / sp_idx in ascending column order) that
 * also writes the same entries in the bank-balanced order to sp_bdata [n x k] fp32 / sp_bidx [n x k] (idx_bytes):
 *   with the rank list Q = (positions 4p+e for e = 0..3, 0 <= p < k/8) followed by (positions 4p+e for
 *   e = 3..0, k/8 <= p < k/4), the row's even columns, in ascending order, take Q[0], Q[1], ... and its odd columns,
 *   in ascending order, Q[k-1], Q[k-2], ...; sp_bdata[r, t] = x[r, sp_bidx[r, t]] (bit copy).
 * Positions t and t + k/2 then hold columns of different parity unless the row has more than k/2 columns of one
 * parity; in the forward's NC = 16 layout such a pair costs a bank conflict, where the column order costs one on
 * ~every read-modify-write instruction.  Pass sp_bdata / sp_bidx to maxk_spgemm_fwd (same Y up to fp32 summation
 * order); the backward keeps sp_idx (its d_sp_data is then in column order).
 *   Errors: as maxk_topk_cbsr; INVALID_ARGUMENT for a NULL sp_bdata / sp_bidx with n_rows > 0; UNSUPPORTED unless
 *   k in {32, 64, 128} and h in {128, 256, 384, 512} with 16-byte aligned rows of x.
 */
maxk_status_t maxk_topk_cbsr_banked(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                    int32_t idx_bytes, float* sp_data, void* sp_idx, float* sp_bdata,
                                    void* sp_bidx, maxk_stream_t stream);

/*
 * Whether the forward on a graph of n_rows rows and nnz edges at (h, k) uses replicated row buffers (its measured
 * default policy): NC = 16 copies in maxk_spgemm_fwd at k >= 32, NC = 8 copies in
 * maxk_spgemm_fwd_pairs at k = 16 — the layouts the bank-balanced copies (maxk_topk_cbsr_banked,
 * maxk_topk_cbsr_pairs_banked) are for.  Host-only, no validation (returns 0 for arguments the forward would
 * reject).  MAXK_FWD_REP=0 / 2 in the environment force the answer as they force the forward.
 */
int32_t maxk_spgemm_fwd_replicated(int64_t n_rows, int64_t nnz, int32_t h, int32_t k);

/*
 * The all-gather fused into the top-k: maxk_topk_cbsr writing each CBSR row to
 * n_dst destinations at once, so the replicas of a row-partitioned layer receive the rank's block straight from
 * the top-k epilogue (peer stores over NVLink for replicas in peers' memory) instead of through a separate
 * all-gather.
 *   sp_data, sp_idx  HOST arrays of n_dst DEVICE pointers, each the first row of this block in one replica
 *                    ([n_rows x k], row stride k; entry 0 is written exactly like maxk_topk_cbsr's outputs)
 *   Other arguments as maxk_topk_cbsr.  The pointers must be dereferenceable from the current device (this
 *   device's memory, or peers' memory mapped into this process, e.g. torch symmetric memory).
 *   Errors: as maxk_topk_cbsr; INVALID_ARGUMENT for n_dst outside [1, 8] or a NULL destination; UNSUPPORTED
 *   unless k in {8, 16, 32, 64} and h in {128, 256} with 16-byte aligned rows of x.
 */
maxk_status_t maxk_topk_cbsr_multi(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                   int32_t idx_bytes, int32_t n_dst, float* const* sp_data, void* const* sp_idx,
                                   maxk_stream_t stream);

/*
 * Debug statistic of the pivot search (NOT the hot path; "median iterations <= 10", PAPER.md:675
 * "less than 10 iterations"): the same selection as maxk_topk_cbsr (identical sp_data / sp_idx), and
 * probes[r] (DEVICE int32 [n_rows], written) = number of pivot probes row r took, plus 1000 when the exact key
 * descent (the fallback for boundary ties, +-Inf, fp32 stalls) decided it.
 * Errors: as maxk_topk_cbsr; UNSUPPORTED unless h in {128, 256, 384, 512} with 16-byte aligned rows and
 * k in {8, 16, 32, 64, 96, 128} (the compile-time kernels of the hot path).
 */
maxk_status_t maxk_topk_cbsr_probe_stats(const float* x, int64_t n_rows, int32_t h, int64_t ld_x, int32_t k,
                                         int32_t idx_bytes, float* sp_data, void* sp_idx, int32_t* probes,
                                         maxk_stream_t stream);

/*
 * Work plan for one CSR graph (the paper's warp-level partition meta-data, §4.1 and
 * PAPER.md:493 §4.2, redesigned as degree-sorted units with hub-row splitting).
 *   row_ptr  DEVICE [n_rows+1] int64 — copied to the host once (this call synchronises `stream`).
 *   nnz      must equal row_ptr[n_rows] - row_ptr[0]
 *   h, k     the feature widths the plan will be used with (sizes the split-row scratch)
 *   out      receives the plan; destroy with maxk_plan_destroy.
 * Errors: INVALID_ARGUMENT (bad sizes, non-monotone row_ptr, nnz mismatch), OUT_OF_MEMORY, CUDA.
 * A plan may serve any number of forward/backward calls on the same graph, ONE CALL AT A TIME, in stream
 * order (it holds device-side ticket counters, reset by each launch's last warp, and the split-row scratch):
 * two calls in flight on different streams with the same plan are undefined (skipped or repeated work
 * units). Use one plan per concurrently running stream. A plan belongs to the device that was current at
 * maxk_plan_create; a call made while another device is current returns INVALID_ARGUMENT.
 */
maxk_status_t maxk_plan_create(const int64_t* row_ptr, int64_t n_rows, int64_t nnz, int32_t h, int32_t k,
                               maxk_stream_t stream, maxk_plan_t** out);
void maxk_plan_destroy(maxk_plan_t* plan);

/*
 * Plan statistics (HOST pointers, any may be NULL): number of work units, number of hub rows split
 * into chunks, chunk length in edges, number of chunk units.  Returns INVALID_ARGUMENT on a NULL plan.
 */
maxk_status_t maxk_plan_info(const maxk_plan_t* plan, int64_t* n_units, int64_t* n_split_rows,
                             int64_t* chunk_edges, int64_t* n_chunk_units);

/*
 * Forward SpGEMM (Eq. 3 left; row-wise product PAPER.md:326; Alg. 1):
 *   y[i, :] = sum_{e in row i} val[e] * densify(sp_data, sp_idx)[col_idx[e], :]
 * y is fully OVERWRITTEN (rows with no edges become 0). fp32 accumulation; per-row summation order
 * is fixed by the plan (deterministic run to run).
 *   row_ptr/col_idx/val  CSR of A (n_rows x n_cols)                        (read)
 *   sp_data, sp_idx      CBSR [n_cols x k]                                  (read)
 *   y                    [n_rows x h], row stride ld_y >= h                  (written)
 *   plan                 from maxk_plan_create on this row_ptr, or NULL (slower plan-free path)
 * Errors: INVALID_ARGUMENT (sizes, widths, ld_y < h, NULL pointers with nonzero extent, plan built
 *         for a different n_rows/nnz or on another device); UNSUPPORTED for h > 4096, k > 1024 or n_cols > INT32_MAX.
 */
maxk_status_t maxk_spgemm_fwd(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                              int64_t n_rows, int64_t n_cols, int64_t nnz,
                              const float* sp_data, const void* sp_idx, int32_t h, int32_t k,
                              int32_t idx_bytes, float* y, int64_t ld_y,
                              const maxk_plan_t* plan, maxk_stream_t stream);

/*
 * maxk_spgemm_fwd reading the CBSR in the pair layout (see maxk_topk_cbsr_pairs): same result, same
 * determinism.  sp_pairs [n_cols x k] (read).  Errors: as maxk_spgemm_fwd; INVALID_ARGUMENT for a misaligned
 * sp_pairs; UNSUPPORTED unless k in {8, 16}.
 */
maxk_status_t maxk_spgemm_fwd_pairs(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                    int64_t n_rows, int64_t n_cols, int64_t nnz, const void* sp_pairs, int32_t h,
                                    int32_t k, float* y, int64_t ld_y, const maxk_plan_t* plan,
                                    maxk_stream_t stream);

/*
 * Backward SSpMM (Eq. 3 right; outer-product form Eq. 4; Alg. 2,
 * PAPER.md:447-468 with line 9 read as d_sp_data[j,t] += A[i,j] * dY[i, sp_idx[j,t]], R8):
 *   d_sp_data[j, t] = sum_{e=(i,j) in A} val[e] * dy[i, sp_idx[j, t]]
 * d_sp_data is fully OVERWRITTEN (zeroed, then accumulated with fp32 reductions in L2; summation
 * order is not deterministic). The mask is the forward's sp_idx, so it is identical by construction.
 *   row_ptr/col_idx/val  CSR of A (n_rows x n_cols), read as the CSC of A^T  (read)
 *   dy                   [n_rows x h], row stride ld_dy >= h                  (read)
 *   sp_idx               [n_cols x k] (the forward pattern)                    (read)
 *   d_sp_data            [n_cols x k] fp32                                     (written)
 * Errors: as maxk_spgemm_fwd.
 */
maxk_status_t maxk_sspmm_bwd(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                             int64_t n_rows, int64_t n_cols, int64_t nnz,
                             const float* dy, int64_t ld_dy, const void* sp_idx, int32_t h, int32_t k,
                             int32_t idx_bytes, float* d_sp_data,
                             const maxk_plan_t* plan, maxk_stream_t stream);

/*
 * Accumulating forms (the multi-GPU comm/compute overlap): identical to
 * maxk_spgemm_fwd / maxk_sspmm_bwd except that the output is NOT overwritten:
 *   maxk_spgemm_fwd_acc:  y[i, :] += sum_{e in row i} val[e] * densify(sp_data, sp_idx)[col_idx[e], :]
 *   maxk_sspmm_bwd_acc:   d_sp_data[j, t] += sum_{e=(i,j)} val[e] * dy[i, sp_idx[j, t]]  (no zero-fill)
 * A rank computes its local-column edges while the CBSR all-gather is in flight and then accumulates the
 * remote-column edges; the sum over the two edge sets equals the single call on the union (fp32 rounding
 * aside). Arguments, layouts and errors as the overwriting calls.
 */
maxk_status_t maxk_spgemm_fwd_acc(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                  int64_t n_rows, int64_t n_cols, int64_t nnz,
                                  const float* sp_data, const void* sp_idx, int32_t h, int32_t k,
                                  int32_t idx_bytes, float* y, int64_t ld_y,
                                  const maxk_plan_t* plan, maxk_stream_t stream);
maxk_status_t maxk_sspmm_bwd_acc(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                 int64_t n_rows, int64_t n_cols, int64_t nnz,
                                 const float* dy, int64_t ld_dy, const void* sp_idx, int32_t h, int32_t k,
                                 int32_t idx_bytes, float* d_sp_data,
                                 const maxk_plan_t* plan, maxk_stream_t stream);

/*
 * The reduce-scatter fused into the backward: maxk_sspmm_bwd whose reductions for
 * CBSR row (slot) j go straight to its owner, d_owner[j / owner_rows] + (j % owner_rows) * k, instead of a local
 * [n_cols x k] partial that a reduce-scatter would then move (peer reductions over NVLink for owners in peers'
 * memory).  Accumulating: every owner zeroes its block before the ranks' calls (they may run concurrently;
 * the fp32 reduction order is not deterministic, as in maxk_sspmm_bwd).
 *   n_owners, owner_rows  n_cols == n_owners * owner_rows (the slot space of DESIGN.md §6), owner_rows < 2^24
 *   d_owner  DEVICE array of n_owners DEVICE pointers, each 16-byte aligned, [owner_rows x k] fp32 (read-modify-
 *            written); dereferenceable from the current device
 *   Other arguments as maxk_sspmm_bwd (d_sp_data is not used).
 *   Errors: as maxk_sspmm_bwd; INVALID_ARGUMENT for a size mismatch or NULL d_owner; UNSUPPORTED for k without a
 *   vector backward (k not in {8, 16, 32, 64, 96, 128, 192, 256}) or misaligned sp_idx.
 */
maxk_status_t maxk_sspmm_bwd_owners(const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                    int64_t n_rows, int64_t n_cols, int64_t nnz, const float* dy, int64_t ld_dy,
                                    const void* sp_idx, int32_t h, int32_t k, int32_t idx_bytes, int32_t n_owners,
                                    int64_t owner_rows, float* const* d_owner, const maxk_plan_t* plan,
                                    maxk_stream_t stream);

/*
 * dst[i] += src[i] for i < n (fp32, DEVICE pointers; f2: the local-target backward partial added to the
 * reduce-scatter result). Errors: INVALID_ARGUMENT for n < 0 or NULL pointers with n > 0.
 */
maxk_status_t maxk_add_f32(float* dst, const float* src, int64_t n, maxk_stream_t stream);

/*
 * MaxK backward scatter: the dense gradient of the MaxK nonlinearity's input.
 * "The feature gradient uses the same sparsity pattern as induced in the forward pass" (PAPER.md:226,
 * §3.1 Def. ii; SPEC.md:141-149 maxk_backward):
 *   dx[r, sp_idx[r, t]] = d_sp_data[r, t] for t < k;  dx[r, c] = 0 for every other column c.
 *   d_sp_data  [n_rows x k] fp32 (e.g. maxk_sspmm_bwd's output)            (read)
 *   sp_idx     [n_rows x k] uint8/uint16, the forward pattern               (read)
 *   dx         [n_rows x h] fp32, row stride ld_dx >= h, fully OVERWRITTEN  (written)
 * Errors: INVALID_ARGUMENT as maxk_topk_cbsr (k, h, idx_bytes, ld, NULL); UNSUPPORTED for h > 4096.
 */
maxk_status_t maxk_cbsr_scatter(const float* d_sp_data, const void* sp_idx, int64_t n_rows, int32_t h, int32_t k,
                                int32_t idx_bytes, float* dx, int64_t ld_dx, maxk_stream_t stream);

/*
 * Eq. 1 in full, fused on the tensor cores: h(X) = max-k (X·W + b) -> CBSR
 * (PAPER.md:228-234).  z = X·W + b is computed with tcgen05 (bf16 x bf16 products accumulated in fp32,
 * in TMEM) and never written to HBM; the selection is the exact top-k of that fp32 z with the same rule as
 * maxk_topk_cbsr (value descending, lower column on ties, -0.0 == +0.0, z bits copied).
 *   x        [n_rows x f_in] bf16 (raw 16-bit patterns), row stride ld_x elements; 16-byte aligned base and
 *            ld_x a multiple of 8 (TMA)                                                         (read)
 *   w_t      [h x f_in] bf16 = W transposed (each output column's weights contiguous), stride ld_w (read)
 *   bias     [h] fp32, or NULL for b = 0                                                         (read)
 *   h        128 or 256;  f_in a multiple of 64 with f_in * h * 2 <= 131072 (W stays in shared memory)
 *   k        1 <= k <= min(h, 64)
 *   sp_data, sp_idx  as maxk_topk_cbsr                                                           (written)
 *   z_out    optional [n_rows x h] fp32, row stride ld_z >= h (a multiple of 4, 16-byte aligned base): receives z
 *            itself (verification) or NULL
 * Errors: INVALID_ARGUMENT (sizes, alignment, NULL pointers, k), UNSUPPORTED (h, f_in, k out of the ranges
 *         above), CUDA (tensor-map encoding or launch failures).
 */
maxk_status_t maxk_linear_topk_cbsr(const void* x, int64_t n_rows, int32_t f_in, int64_t ld_x, const void* w_t,
                                    int64_t ld_w, const float* bias, int32_t h, int32_t k, int32_t idx_bytes,
                                    float* sp_data, void* sp_idx, float* z_out, int64_t ld_z, maxk_stream_t stream);

/* Human-readable name of a status. Never NULL. */
/*
 * Debug-only validation of the input-VALUE contract the layer calls trust (never called on the hot path;
 * each call synchronises `stream` once and allocates a few bytes):
 *   maxk_validate_csr:  bad_rows = rows with row_ptr[i+1] < row_ptr[i]; bad_cols = edges with col_idx outside
 *                       [0, n_cols). col_idx is indexed absolutely (row_ptr[0] may be nonzero).
 *   maxk_validate_cbsr: bad_rows = CBSR rows whose k indices are not strictly ascending or not < h (SPEC.md:110,
 *                       169) — the precondition of maxk_spgemm_fwd / maxk_sspmm_bwd / maxk_cbsr_scatter.
 * Output counts are HOST pointers (may be NULL). Errors: INVALID_ARGUMENT, CUDA.
 */
maxk_status_t maxk_validate_csr(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols,
                                maxk_stream_t stream, int64_t* bad_rows, int64_t* bad_cols);
maxk_status_t maxk_validate_cbsr(const void* sp_idx, int64_t n_rows, int32_t h, int32_t k, int32_t idx_bytes,
                                 maxk_stream_t stream, int64_t* bad_rows);

const char* maxk_status_string(maxk_status_t s);
/* Thread-local detail of the last error returned on this thread ("" if none). Never NULL. */
const char* maxk_last_error_detail(void);
/* Number of kernels this library has launched in this process (monotone; for launch accounting). */
uint64_t maxk_launch_count(void);
/* Library version string, e.g. "maxk-b200 0.1 sm_100a". */
const char* maxk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MAXK_H_ */
