// tg_adamw.cu -- the optimizer step of the LM head ("in LLM
// terms: LM-head backward GEMM plus a fused AdamW"), the LLM-scale counterpart of
// algorithms.apply_update (algorithms.py:329-348; tg_update.cu keeps its SGD).
//
// torch.optim.AdamW semantics (decoupled weight decay), one HBM pass:
//     m = m + (1 - b1) (g - m)                  (torch: exp_avg.lerp_(g, 1 - b1))
//     v = b2 v + (1 - b2) g^2
//     p = p (1 - lr wd) - lr / (1 - b1^t) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)
// p bf16 or fp32 with a row pitch (a slice of the LM head), g bf16 or fp32 (the
// tcgen05 d W of tg_lmhead_grad_*), m / v fp32 contiguous.  Per bf16 parameter
// 22 bytes of HBM traffic (p read + write 4, g 2, m 8, v 8): HBM-bound, so the
// kernel moves 4-parameter units (every warp access one contiguous span), 4
// units per thread in flight, over a persistent grid of whole waves.  As apply_update refuses a non-finite
// gradient before writing (algorithms.py:337-338), a caller-supplied status
// word turns on a read-only pass over g first, and the update leaves
// everything untouched when it found one (status 1).
#include "tg_common.cuh"

#include <cmath>

namespace tg {

struct AdamwParams {
  void* param;
  int pdtype;
  int64_t ld_param;
  const void* grad;
  int gdtype;
  int64_t ld_grad;
  float* m;
  float* v;
  int64_t rows, cols;
  float lr, b1, b2, eps, decay;  // decay = 1 - lr wd
  float step_size;                // lr / (1 - b1^t)
  float rbc2;                     // 1 / sqrt(1 - b2^t)
  const int32_t* status;          // non-null: skip the update when *status != 0
};

// 4 consecutive elements of a row as fp32 (an 8-byte bf16 vector or a float4):
// with 4-element units every access of a warp is one contiguous, fully used
// span (param / grad 256 or 512 B, each moment 512 B)
template <typename T>
__device__ __forceinline__ void load4(const void* base, int64_t off, float (&x)[4]) {
  if constexpr (sizeof(T) == 2) {
    const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(base) + off);
    x[0] = __uint_as_float(u.x << 16);
    x[1] = __uint_as_float(u.x & 0xffff0000u);
    x[2] = __uint_as_float(u.y << 16);
    x[3] = __uint_as_float(u.y & 0xffff0000u);
  } else {
    const float4 a = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  }
}

template <typename T>
__device__ __forceinline__ void store4(void* base, int64_t off, const float (&x)[4]) {
  if constexpr (sizeof(T) == 2) {
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(base) + off) =
        make_uint2(Vec<bf16_t>::pack2(x[0], x[1]), Vec<bf16_t>::pack2(x[2], x[3]));
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + off) =
        make_float4(x[0], x[1], x[2], x[3]);
  }
}

__device__ __forceinline__ float adamw_one(float& p, float g, float& m, float& v,
                                           const AdamwParams& a) {
  m = fmaf(1.f - a.b1, g - m, m);
  v = fmaf((1.f - a.b2) * g, g, a.b2 * v);
  const float denom = sqrtf(v) * a.rbc2 + a.eps;
  p = p * a.decay - a.step_size * (m / denom);
  return p;
}

// one 4-parameter unit: the loads of all units of a batch are issued before
// any math (memory-level parallelism), then update and stores
struct AdamwUnit {
  float p[4], g[4], m[4], v[4];
};

template <typename TP, typename TG>
__device__ __forceinline__ void unit_load(AdamwUnit& u, const AdamwParams& a, int64_t r,
                                          int64_t col) {
  load4<TP>(a.param, r * a.ld_param + col, u.p);
  load4<TG>(a.grad, r * a.ld_grad + col, u.g);
  load4<float>(a.m, r * a.cols + col, u.m);
  load4<float>(a.v, r * a.cols + col, u.v);
}

template <typename TP>
__device__ __forceinline__ void unit_store(const AdamwUnit& u, const AdamwParams& a, int64_t r,
                                           int64_t col) {
  store4<TP>(a.param, r * a.ld_param + col, u.p);
  store4<float>(a.m, r * a.cols + col, u.m);
  store4<float>(a.v, r * a.cols + col, u.v);
}

// kVec: cols % 4 == 0 and 8 / 16-byte aligned rows -> 4-element units, kU units
// per thread and iteration (grid-stride).  Measured on B200 (LM head 151,936 x
// 1,536, profiles/r02_adamw.txt): bf16 parameters 2 units (0.95 of the copy
// peak; 4: 0.67, 8: 0.40), fp32 parameters 4 units (0.94; 2: 0.89, 8: 0.78).
template <typename TP>
constexpr int adamw_units() {
#ifdef TG_ADAMW_U
  return TG_ADAMW_U;
#else
  return sizeof(TP) == 2 ? 2 : 4;
#endif
}

template <typename TP, typename TG, bool kVec>
__global__ void __launch_bounds__(256) k_adamw(const AdamwParams a) {
  if (a.status && *a.status != 0) return;  // refused: nothing is written
  constexpr int kAdamwU = adamw_units<TP>();
  const int64_t per_row = kVec ? a.cols / 4 : a.cols;
  const int64_t n = a.rows * per_row;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if constexpr (kVec) {
    for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n;
         i0 += kAdamwU * stride) {
      AdamwUnit u[kAdamwU];
#pragma unroll
      for (int k = 0; k < kAdamwU; ++k) {
        const int64_t i = i0 + k * stride;
        if (i < n) {
          const int64_t r = i / per_row;
          unit_load<TP, TG>(u[k], a, r, (i - r * per_row) * 4);
        }
      }
#pragma unroll
      for (int k = 0; k < kAdamwU; ++k) {
        const int64_t i = i0 + k * stride;
        if (i < n) {
#pragma unroll
          for (int e = 0; e < 4; ++e) adamw_one(u[k].p[e], u[k].g[e], u[k].m[e], u[k].v[e], a);
          const int64_t r = i / per_row;
          unit_store<TP>(u[k], a, r, (i - r * per_row) * 4);
        }
      }
    }
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
      const int64_t r = i / per_row, c = i - r * per_row;
      float p = Vec<TP>::load1(reinterpret_cast<const char*>(a.param) +
                                   r * a.ld_param * int64_t(sizeof(TP)), c);
      const float g = Vec<TG>::load1(reinterpret_cast<const char*>(a.grad) +
                                         r * a.ld_grad * int64_t(sizeof(TG)), c);
      float m = a.m[r * a.cols + c], v = a.v[r * a.cols + c];
      adamw_one(p, g, m, v, a);
      Vec<TP>::store1(reinterpret_cast<char*>(a.param) + r * a.ld_param * int64_t(sizeof(TP)), c,
                      p);
      a.m[r * a.cols + c] = m;
      a.v[r * a.cols + c] = v;
    }
  }
}

template <typename TG, bool kVec>
__global__ void __launch_bounds__(256) k_adamw_check(const AdamwParams a, int32_t* status) {
  int bad = 0;
  const int64_t per_row = kVec ? a.cols / 4 : a.cols;
  const int64_t n = a.rows * per_row;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, c = i - r * per_row;
    if constexpr (kVec) {
      float g[4];
      load4<TG>(a.grad, r * a.ld_grad + c * 4, g);
#pragma unroll
      for (int k = 0; k < 4; ++k) bad |= !isfinite(g[k]);
    } else {
      const float g = Vec<TG>::load1(reinterpret_cast<const char*>(a.grad) +
                                         r * a.ld_grad * int64_t(sizeof(TG)), c);
      bad |= !isfinite(g);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, 1);
}

// persistent grid: the resident CTAs of the kernel (occupancy query), at most
// one per 256 units
template <typename K>
static int resident_grid(K kernel, int n_sms, int64_t units) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t grid = (units + 255) / 256;
  const int64_t cap = int64_t(n_sms > 0 ? n_sms : 148) * per_sm;
  if (grid > cap) grid = cap;
  return grid < 1 ? 1 : int(grid);
}

template <typename TG>
static void check_launch(const AdamwParams& a, bool vec, int64_t units, int n_sms,
                         int32_t* status, cudaStream_t st) {
  if (vec)
    k_adamw_check<TG, true><<<resident_grid(k_adamw_check<TG, true>, n_sms, units), 256, 0, st>>>(
        a, status);
  else
    k_adamw_check<TG, false><<<resident_grid(k_adamw_check<TG, false>, n_sms, units), 256, 0,
                                st>>>(a, status);
}

template <typename TP, typename TG>
static void adamw_launch(const AdamwParams& a, bool vec, int64_t units, int n_sms,
                         cudaStream_t st) {
  if (vec)
    k_adamw<TP, TG, true><<<resident_grid(k_adamw<TP, TG, true>, n_sms, units), 256, 0, st>>>(a);
  else
    k_adamw<TP, TG, false><<<resident_grid(k_adamw<TP, TG, false>, n_sms, units), 256, 0, st>>>(
        a);
}

cudaError_t launch_adamw(void* param, int pdtype, int64_t ld_param, const void* grad, int gdtype,
                         int64_t ld_grad, float* m, float* v, int64_t rows, int64_t cols,
                         double lr, double b1, double b2, double eps, double wd, int64_t step,
                         int32_t* status, int n_sms, cudaStream_t st, int* n_launches) {
  AdamwParams a;
  a.param = param;
  a.pdtype = pdtype;
  a.ld_param = ld_param;
  a.grad = grad;
  a.gdtype = gdtype;
  a.ld_grad = ld_grad;
  a.m = m;
  a.v = v;
  a.rows = rows;
  a.cols = cols;
  a.lr = float(lr);
  a.b1 = float(b1);
  a.b2 = float(b2);
  a.eps = float(eps);
  a.decay = float(1.0 - lr * wd);
  a.step_size = float(lr / (1.0 - std::pow(b1, double(step))));
  a.rbc2 = float(1.0 / std::sqrt(1.0 - std::pow(b2, double(step))));
  a.status = status;
  *n_launches = 0;
  const int esp = pdtype == TG_DTYPE_BF16 ? 2 : 4, esg = gdtype == TG_DTYPE_BF16 ? 2 : 4;
  // 4-element units: 4 E bytes per param / grad access (8 B bf16, 16 B fp32)
  const bool vec = cols % 4 == 0 && (ld_param * esp) % (4 * esp) == 0 &&
                   (ld_grad * esg) % (4 * esg) == 0 &&
                   reinterpret_cast<uintptr_t>(param) % (4 * esp) == 0 &&
                   reinterpret_cast<uintptr_t>(grad) % (4 * esg) == 0 &&
                   reinterpret_cast<uintptr_t>(m) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(v) % 16 == 0;
  const int64_t units = rows * (vec ? cols / 4 : cols);
  if (status) {
    cudaMemsetAsync(status, 0, sizeof(int32_t), st);
    if (gdtype == TG_DTYPE_BF16)
      check_launch<bf16_t>(a, vec, units, n_sms, status, st);
    else
      check_launch<float>(a, vec, units, n_sms, status, st);
    ++*n_launches;
  }
  if (pdtype == TG_DTYPE_BF16) {
    if (gdtype == TG_DTYPE_BF16)
      adamw_launch<bf16_t, bf16_t>(a, vec, units, n_sms, st);
    else
      adamw_launch<bf16_t, float>(a, vec, units, n_sms, st);
  } else {
    if (gdtype == TG_DTYPE_BF16)
      adamw_launch<float, bf16_t>(a, vec, units, n_sms, st);
    else
      adamw_launch<float, float>(a, vec, units, n_sms, st);
  }
  ++*n_launches;
  return cudaGetLastError();
}

}  // namespace tg
