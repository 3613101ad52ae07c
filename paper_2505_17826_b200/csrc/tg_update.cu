// tg_update.cu -- the optimizer step after the loss path:
// algorithms.apply_update (algorithms.py:329-348) on the device.
//
//   theta[s, :] -= lr * sum_{rows r with state(r) = s} dlogits[r, :]
//
// for the bucketed logits table of the reference policy (policy.py:59-94),
// whose per-token gradient rows are the dlogits rows the loss kernels wrote
// (row r scored table row state(r) through row_index).  Semantics follow the
// reference exactly where it is observable:
//  * a non-finite gradient is refused before anything is written
//    (algorithms.py:337-338): k_update_check scans the gradient rows and sets
//    a device status word that k_update_apply reads first;
//  * a state outside [0, S) is refused (algorithms.py:341-342), status 2;
//  * per state the rows are summed in f64, in row order (the order
//    SparseGrad.add_row / axpy accumulate them, policy.py:215-250), and the
//    table is updated once: deterministic, no atomics.
// The caller passes the rows grouped by state (CSR: state_offsets over
// row_order, built on the host from the FNV states it already holds).
//
//   k_update_check  CTA per touched gradient row (grid-stride): finiteness + state range
//   k_update_apply  CTA per (state, 1024-column block): f64 sums over the
//                   state's rows, then one read-modify-write of the table slice
#include "tg_common.cuh"
#include "tg_rowcoef.cuh"

namespace tg {

struct UpdateParams {
  float* table;               // [S, ld_table] fp32
  int64_t ld_table, n_states, vocab;
  const void* grad;           // [*, ld_grad] bf16 or fp32
  int dtype;
  int64_t ld_grad;
  const int64_t* state_ids;   // [n_touched]
  const int64_t* state_offsets;  // [n_touched + 1] into row_order
  const int64_t* row_order;   // [n_rows] gradient rows grouped by state, row order within
  int64_t n_touched;
  double lr;
  int32_t* status;            // [1] 0 ok, 1 non-finite gradient, 2 state out of range
};

template <typename T>
__device__ __forceinline__ float grad_at(const UpdateParams& p, int64_t r, int64_t v) {
  return Vec<T>::load1(reinterpret_cast<const char*>(p.grad) + r * p.ld_grad * int64_t(sizeof(T)),
                       v);
}

template <typename T>
__global__ void k_update_check(const UpdateParams p) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  int mine = 0;
  // states first (cheap), then every gradient element of the touched rows
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n_touched;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = p.state_ids[i];
    if (s < 0 || s >= p.n_states) mine |= 2;
  }
  const int64_t n_rows = p.n_touched > 0 ? p.state_offsets[p.n_touched] : 0;
  for (int64_t j = blockIdx.x; j < n_rows; j += gridDim.x) {
    const int64_t r = p.row_order[j];
    for (int64_t v = threadIdx.x; v < p.vocab; v += blockDim.x)
      if (!finite_f(grad_at<T>(p, r, v))) mine |= 1;
  }
  if (mine) atomicOr(&bad, mine);
  __syncthreads();
  if (threadIdx.x == 0 && bad) atomicOr(p.status, bad);
}

template <typename T>
__global__ void __launch_bounds__(256) k_update_apply(const UpdateParams p) {
  if (*p.status != 0) return;  // refused: nothing is written
  const int64_t st = blockIdx.y;
  const int64_t s = p.state_ids[st];
  const int64_t r0 = p.state_offsets[st], r1 = p.state_offsets[st + 1];
  const int64_t v0 = int64_t(blockIdx.x) * 1024;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t j = r0; j < r1; ++j) {  // row order: the reference's accumulation order
    const int64_t r = p.row_order[j];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t v = v0 + threadIdx.x + 256 * k;
      if (v < p.vocab) acc[k] += double(grad_at<T>(p, r, v));
    }
  }
  float* row = p.table + s * p.ld_table;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t v = v0 + threadIdx.x + 256 * k;
    if (v < p.vocab) row[v] = float(double(row[v]) - p.lr * acc[k]);
  }
}

cudaError_t launch_update(float* table, int64_t ld_table, int64_t n_states, int64_t vocab,
                          const void* grad, int dtype, int64_t ld_grad, const int64_t* state_ids,
                          const int64_t* state_offsets, const int64_t* row_order,
                          int64_t n_touched, int64_t n_rows, double lr, int32_t* status,
                          cudaStream_t stream) {
  UpdateParams p;
  p.table = table;
  p.ld_table = ld_table;
  p.n_states = n_states;
  p.vocab = vocab;
  p.grad = grad;
  p.dtype = dtype;
  p.ld_grad = ld_grad;
  p.state_ids = state_ids;
  p.state_offsets = state_offsets;
  p.row_order = row_order;
  p.n_touched = n_touched;
  p.lr = lr;
  p.status = status;
  cudaMemsetAsync(status, 0, sizeof(int32_t), stream);
  if (n_touched == 0) return cudaGetLastError();
  const int check_grid = int(n_rows < 4096 ? (n_rows > 0 ? n_rows : 1) : 4096);
  const dim3 apply_grid(unsigned((vocab + 1023) / 1024), unsigned(n_touched));
  if (dtype == TG_DTYPE_BF16) {
    k_update_check<bf16_t><<<check_grid, 256, 0, stream>>>(p);
    k_update_apply<bf16_t><<<apply_grid, 256, 0, stream>>>(p);
  } else {
    k_update_check<float><<<check_grid, 256, 0, stream>>>(p);
    k_update_apply<float><<<apply_grid, 256, 0, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace tg
