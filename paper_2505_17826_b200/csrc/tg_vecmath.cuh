// tg_vecmath.cuh -- packed element math shared by the row kernels (sm_100a).
//
// 16-byte vectors of 8 bf16 / 4 fp32 logits; packed bf16x2 max (clamp of
// -inf, vector max), packed fp32x2 FFMA2 / FADD2 / FMUL2 arithmetic, MUFU ex2,
// the lazily-rescaled online (max, sum e, sum e z) accumulator and the dz
// epilogue p (a + h z).
#pragma once

#include "tg_common.cuh"

namespace tg {

// ---- packed-element helpers (bf16: 8 per vector, fp32: 4 per vector) --------

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

constexpr uint32_t kBf16NegBig2 = 0xF149F149u;  // (-1.0e30, -1.0e30) as bf16x2
constexpr uint32_t kF32NegBig = 0xF149F2CAu;    // -1.0e30f
constexpr float kNegBig = -1.0e30f;

template <typename T>
struct Pk;

template <>
struct Pk<bf16_t> {
  // clamp -inf (masked vocabulary) to -1e30 so p = 0 without NaN from 0 * -inf
  __device__ __forceinline__ static void clamp(uint4& u) {
    u.x = bmax2(u.x, kBf16NegBig2);
    u.y = bmax2(u.y, kBf16NegBig2);
    u.z = bmax2(u.z, kBf16NegBig2);
    u.w = bmax2(u.w, kBf16NegBig2);
  }
  __device__ __forceinline__ static uint4 neutral() {
    return make_uint4(kBf16NegBig2, kBf16NegBig2, kBf16NegBig2, kBf16NegBig2);
  }
  __device__ __forceinline__ static uint32_t pmax(const uint4& u) {
    return bmax2(bmax2(u.x, u.y), bmax2(u.z, u.w));
  }
  __device__ __forceinline__ static float hmax(uint32_t m) {
    return fmaxf(__uint_as_float(m << 16), __uint_as_float(m & 0xffff0000u));
  }
  __device__ __forceinline__ static float vmax(const uint4& u) { return hmax(pmax(u)); }
  // elements e >= n of the vector become -1e30 (columns past V)
  __device__ __forceinline__ static void mask_from(uint4& u, int n) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e >= n) {
        const uint32_t keep = (e & 1) ? 0x0000ffffu : 0xffff0000u;
        const uint32_t put = (e & 1) ? 0xF1490000u : 0x0000F149u;
        w[e >> 1] = (w[e >> 1] & keep) | put;
      }
  }
  __device__ __forceinline__ static float elem(const uint4& u, int e) {
    const uint32_t w = (e >> 1) == 0 ? u.x : (e >> 1) == 1 ? u.y : (e >> 1) == 2 ? u.z : u.w;
    return (e & 1) ? __uint_as_float(w & 0xffff0000u) : __uint_as_float(w << 16);
  }
};

template <>
struct Pk<float> {
  __device__ __forceinline__ static void clamp(uint4& u) {
    u.x = __float_as_uint(fmaxf(__uint_as_float(u.x), kNegBig));
    u.y = __float_as_uint(fmaxf(__uint_as_float(u.y), kNegBig));
    u.z = __float_as_uint(fmaxf(__uint_as_float(u.z), kNegBig));
    u.w = __float_as_uint(fmaxf(__uint_as_float(u.w), kNegBig));
  }
  __device__ __forceinline__ static uint4 neutral() {
    return make_uint4(kF32NegBig, kF32NegBig, kF32NegBig, kF32NegBig);
  }
  __device__ __forceinline__ static float vmax(const uint4& u) {
    return fmaxf(fmaxf(__uint_as_float(u.x), __uint_as_float(u.y)),
                 fmaxf(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  __device__ __forceinline__ static void mask_from(uint4& u, int n) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e >= n) w[e] = kF32NegBig;
  }
  __device__ __forceinline__ static float elem(const uint4& u, int e) {
    return __uint_as_float(e == 0 ? u.x : e == 1 ? u.y : e == 2 ? u.z : u.w);
  }
};

// max over N vectors
template <typename T, int N>
__device__ __forceinline__ float group_max(const uint4 (&u)[N]) {
  if constexpr (sizeof(T) == 2) {
    uint32_t m = Pk<bf16_t>::pmax(u[0]);
#pragma unroll
    for (int g = 1; g < N; ++g) m = bmax2(m, Pk<bf16_t>::pmax(u[g]));
    return Pk<bf16_t>::hmax(m);
  } else {
    float m = Pk<float>::vmax(u[0]);
#pragma unroll
    for (int g = 1; g < N; ++g) m = fmaxf(m, Pk<float>::vmax(u[g]));
    return m;
  }
}

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100a) -------------

__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// the two elements of 32-bit word w of a vector, as an fp32x2 pair
template <typename T>
__device__ __forceinline__ uint64_t pair(const uint4& u, int w);
template <>
__device__ __forceinline__ uint64_t pair<bf16_t>(const uint4& u, int w) {
  const uint32_t x = w == 0 ? u.x : w == 1 ? u.y : w == 2 ? u.z : u.w;
  return pk2(__uint_as_float(x << 16), __uint_as_float(x & 0xffff0000u));
}
template <>
__device__ __forceinline__ uint64_t pair<float>(const uint4& u, int w) {
  return w == 0 ? pk2(__uint_as_float(u.x), __uint_as_float(u.y))
                : pk2(__uint_as_float(u.z), __uint_as_float(u.w));
}
__device__ __forceinline__ uint64_t ex2x2(uint64_t a) {
  float a0, a1;
  upk2(a, a0, a1);
  return pk2(ex2(a0), ex2(a1));
}

// Phase-1 accumulators as fp32x2 lanes (merged into Online at the end).
// The running max m is updated lazily: terms use p = 2^((x - m) log2e), which
// stays finite while x <= m + kSlack, so the rescale only runs when a vector
// max exceeds m by more than kSlack (a handful of times per row).  Sums of
// < 2^31 terms of <= e^kSlack cannot overflow fp32.
constexpr float kSlack = 16.0f;

struct Acc2 {
  float m;
  uint64_t nm2;  // (-m log2e, -m log2e)
  uint64_t s2, t2;
};

__device__ __forceinline__ void rescale(Acc2& acc, float vmax) {
  if (vmax > acc.m) {
    const float sc = ex2((acc.m - vmax) * kLog2e);  // m = -inf -> 0
    const uint64_t sc2 = pk2(sc, sc);
    acc.s2 = mul2(acc.s2, sc2);
    acc.t2 = mul2(acc.t2, sc2);
    acc.m = vmax;
    const float nmL = -vmax * kLog2e;
    acc.nm2 = pk2(nmL, nmL);
  }
}

template <typename T>
__device__ __forceinline__ void accumulate(Acc2& acc, const uint4& u) {
  const uint64_t l2e2 = pk2(kLog2e, kLog2e);
#pragma unroll
  for (int w = 0; w < Vec<T>::N / 2; ++w) {
    const uint64_t x = pair<T>(u, w);
    const uint64_t p = ex2x2(fma2(x, l2e2, acc.nm2));
    acc.s2 = add2(acc.s2, p);
    acc.t2 = fma2(p, x, acc.t2);
  }
}

// dz of one vector: p * (a + hz * z), p = 2^(z log2e - lse log2e).  Without the
// entropy term (kHasH = false) -inf logits need no clamp: p = 0 exactly.
template <typename T, bool kHasH>
__device__ __forceinline__ void dz_vec(uint4 u, float (&d)[Vec<T>::N], uint64_t nl2, uint64_t av2,
                                       uint64_t hz2) {
  const uint64_t l2e2 = pk2(kLog2e, kLog2e);
  if (kHasH) Pk<T>::clamp(u);
#pragma unroll
  for (int w = 0; w < Vec<T>::N / 2; ++w) {
    const uint64_t x = pair<T>(u, w);
    const uint64_t p = ex2x2(fma2(x, l2e2, nl2));
    const uint64_t r = kHasH ? mul2(p, fma2(hz2, x, av2)) : mul2(p, av2);
    upk2(r, d[2 * w], d[2 * w + 1]);
  }
}

}  // namespace tg
