// tg_common.cuh -- device helpers shared by the RFT loss kernels (sm_100a only).
//
// PTX wrappers for mbarriers, 1-D bulk TMA (cp.async.bulk), cluster DSMEM
// (mapa / st.async), MUFU ex2, bf16x2 pack/unpack, plus the kernel parameter
// block (a flattened TgBatch + TgConfig + TgOut + workspace carve-up).
#pragma once

#include <stdlib.h>

#include <cuda_runtime.h>
#include <stdint.h>

#include "tg_loss.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

namespace tg {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kClampLow = -1e30f;  // finite stand-in for -inf logits in products

// ---------------------------------------------------------------------------
// kernel parameter block

struct KParams {
  // batch
  const void* logits;
  const int64_t* row_index;
  const void* anchor;
  int64_t n_rows, vocab, ld, ld_anchor, ld_out;
  int32_t dtype, n_seqs, n_groups, pad0;
  const int32_t* target;
  const float* old_lp;
  const float* ref_lp;
  const int32_t* seq_off;
  const int32_t* grp_off;
  const float* reward;
  const float* seq_ref_lp;
  const float* advantage;
  const uint8_t* seq_kind;
  const float* pg_coef;  // TG_PG_GIVEN: caller's per-row -d l / d lp and l
  const float* pg_loss;
  // outputs (never null after tg_api resolves them to workspace)
  void* dz;
  float* lp;
  float* ent;
  float* lse;
  float* seq_lp;
  float* seq_adv;
  double* stats;
  // workspace
  float* sA;          // [B] advantage (RL) / coupled coefficient
  float* sW;          // [B] aggregation weight
  float* sK;          // [B] size of the sequence's group
  double* sLP;        // [B] sum of lp over the sequence
  double* sRef;       // [B] resolved sequence reference logprob
  double* gF;         // [G * 4] per-group: mean_reward, baseline, loss, aux (rl count / margin)
  float* rS;          // [T] s_t   (two-pass route)
  float* rA;          // [T] a_t   (two-pass route: p * (a + hz*z - ca*za) - s*[v=y])
  float* rHz;         // [T] coefficient of z
  float* rCa;         // [T] coefficient of za (anchor)
  float* rLseQ;       // [T] anchor log-sum-exp
  float* rAkl;        // [T] anchor KL per row
  double* partials;   // [n_partials * TG_NSTAT]
  int64_t* counts;    // [4]: RL rows, RL seqs, SFT seqs, invalid
  int32_t n_partials, pad1;
  // config
  int32_t adv, pg, kl, entf, agg, flags;
  float tau, clip_lo, clip_hi, clip_c, kl_coef, ent_coef, std_eps, sft_w, anchor_beta, dpo_beta,
      agg_norm;
  int64_t n_tok_g, n_seq_g, n_sft_g;
};

// ---------------------------------------------------------------------------
// scalar math

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// online (max, sum e^{z-m}, sum e^{z-m} z) partial; merging is associative.
struct Online {
  float m, s, t;
};

__device__ __forceinline__ Online online_merge(Online a, Online b) {
  const float m = fmaxf(a.m, b.m);
  if (m == kNegInf) return {kNegInf, 0.f, 0.f};
  const float fa = ex2((a.m - m) * kLog2e);  // a.m = -inf -> 0
  const float fb = ex2((b.m - m) * kLog2e);
  return {m, a.s * fa + b.s * fb, a.t * fa + b.t * fb};
}

__device__ __forceinline__ Online warp_merge(Online o) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    Online x;
    x.m = __shfl_xor_sync(0xffffffffu, o.m, d);
    x.s = __shfl_xor_sync(0xffffffffu, o.s, d);
    x.t = __shfl_xor_sync(0xffffffffu, o.t, d);
    o = online_merge(o, x);
  }
  return o;
}

// merge of the partials held by lanes [0, N) (the others hold the neutral
// element): log2(next_pow2(N)) butterfly levels instead of five; lane 0 gets the total
template <int N>
__device__ __forceinline__ Online warp_merge_first(Online o) {
  constexpr int top = N > 16 ? 16 : N > 8 ? 8 : N > 4 ? 4 : N > 2 ? 2 : 1;
#pragma unroll
  for (int d = top; d >= 1; d >>= 1) {
    if (d >= N && d > 1) continue;
    Online x;
    x.m = __shfl_xor_sync(0xffffffffu, o.m, d);
    x.s = __shfl_xor_sync(0xffffffffu, o.s, d);
    x.t = __shfl_xor_sync(0xffffffffu, o.t, d);
    o = online_merge(o, x);
  }
  return o;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// ---------------------------------------------------------------------------
// element packing: one 16-byte vector = 8 bf16 or 4 fp32

template <typename T>
struct Vec;

struct bf16_t {
  uint16_t bits;
};

template <>
struct Vec<bf16_t> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void unpack(const uint4& u, float (&x)[8]) {
    x[0] = __uint_as_float(u.x << 16);
    x[1] = __uint_as_float(u.x & 0xffff0000u);
    x[2] = __uint_as_float(u.y << 16);
    x[3] = __uint_as_float(u.y & 0xffff0000u);
    x[4] = __uint_as_float(u.z << 16);
    x[5] = __uint_as_float(u.z & 0xffff0000u);
    x[6] = __uint_as_float(u.w << 16);
    x[7] = __uint_as_float(u.w & 0xffff0000u);
  }
  __device__ __forceinline__ static uint32_t pack2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  __device__ __forceinline__ static uint4 pack(const float (&x)[8]) {
    return make_uint4(pack2(x[0], x[1]), pack2(x[2], x[3]), pack2(x[4], x[5]), pack2(x[6], x[7]));
  }
  __device__ __forceinline__ static float load1(const void* base, int64_t i) {
    return __uint_as_float(uint32_t(reinterpret_cast<const uint16_t*>(base)[i]) << 16);
  }
  __device__ __forceinline__ static void store1(void* base, int64_t i, float v) {
    reinterpret_cast<uint16_t*>(base)[i] = uint16_t(pack2(v, 0.f) & 0xffffu);
  }
};

template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void unpack(const uint4& u, float (&x)[4]) {
    x[0] = __uint_as_float(u.x);
    x[1] = __uint_as_float(u.y);
    x[2] = __uint_as_float(u.z);
    x[3] = __uint_as_float(u.w);
  }
  __device__ __forceinline__ static uint4 pack(const float (&x)[4]) {
    return make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]),
                      __float_as_uint(x[3]));
  }
  __device__ __forceinline__ static float load1(const void* base, int64_t i) {
    return reinterpret_cast<const float*>(base)[i];
  }
  __device__ __forceinline__ static void store1(void* base, int64_t i, float v) {
    reinterpret_cast<float*>(base)[i] = v;
  }
};

template <typename T>
constexpr int elem_bytes() {
  return sizeof(T) == 2 ? 2 : 4;
}

// ---------------------------------------------------------------------------
// global memory: streaming 128-bit access

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// shared memory, mbarrier, bulk TMA, cluster

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// Run-time A/B switches (TG_FUSED_CL, TG_FUSED_IMPL, TG_FWD_TMA, ...) exist only
// in the A/B build variant (`_build --variant=ab`, libtg_loss_ab.so); the
// product library always takes the measured defaults.
#ifdef TG_AB_SWITCHES
inline int ab_env(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}
#else
inline int ab_env(const char*, int dflt) { return dflt; }
#endif

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor in the stream still runs; pdl_wait() blocks the calling thread
// until the predecessor grid has completed and its writes are visible (a
// no-op without the attribute); pdl_trigger() lets this grid's dependents be
// scheduled once every CTA has issued it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

// try_wait with a suspend-time hint: the warp sleeps until the phase completes
// (or the hint expires) instead of re-issuing the poll, so idle waiters
// (producer, epilogue warp) do not steal issue slots from the math warps.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

template <int kSleep>
__device__ __forceinline__ void mbar_wait_cluster_sleep(uint32_t addr, uint32_t parity) {
  while (!mbar_try_wait_cluster(addr, parity)) {
    if constexpr (kSleep > 0) __nanosleep(kSleep);
  }
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait_cluster(a, parity)) {
  }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier (TMA engine).
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}

// 16-byte remote store into a peer CTA's shared memory, completing tx bytes on
// the peer's mbarrier (DSMEM, asynchronous).
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float a, float b, float c,
                                            float d, uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::
          "r"(remote_addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(remote_bar)
      : "memory");
}

// 4-byte remote store completing tx bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float a, uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
          remote_addr),
      "r"(__float_as_uint(a)), "r"(remote_bar)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tg
