// tg_fused_tma.cu -- K1: fused single-pass logprob + loss + dlogits over [T, V] logits.
//
// Replaces, per trainable row, policy.logprob (policy.py:194-212),
// policy.grad_logprob (policy.py:253-270) and the per-variant axpy of the
// loss's coefficient (algorithms.py:240-242, 263-266) -- plus the north_star
// PPO clip / KL / entropy terms -- with one read of the row from HBM and one
// write of d loss / d logits (4V bytes per row, the HBM roofline minimum).
//
// Design (B200-first):
//  * A thread-block cluster of CL CTAs (CL = 1 for V <= ~98k bf16, 2 for
//    Qwen's 151,936, 4 for fp32 at that vocabulary) owns one row at a time;
//    CTA rank r owns a contiguous column slice of the row, read from HBM
//    exactly once: a producer warp streams it into a 7-slot shared-memory ring
//    (32 KB chunks, 224 KB) with 1-D bulk TMA (cp.async.bulk ...
//    mbarrier::complete_tx), a full / empty mbarrier pair per slot.
//  * 16 consumer warps (4 per SM sub-partition), four 16-byte vectors per
//    thread per chunk.  Phase 1 (as chunks land): online sum-exp / sum p*z in
//    packed fp32x2 arithmetic (FFMA2 / FADD2) with MUFU ex2, speculatively
//    against the warp's reference max (clamp / max / rescale only when the
//    chunk's sums are unsafe).  Each thread copies its raw chunk data into its
//    own TMEM lane (tcgen05.st) and the shared-memory slot is released at once:
//    the row slices stay resident in the otherwise idle TMEM, the ring is pure
//    read-ahead.  Each warp posts its partial to every CTA of the cluster
//    (DSMEM st.async completing tx bytes on the peers' partials barrier).
//  * A dedicated epilogue warp merges all CL x 16 partials in a fixed lane
//    order (bit-identical lse on every CTA), takes the target logit it read
//    from global memory ahead of the wait, evaluates the registry epilogue
//    (tg_rowcoef.cuh) and broadcasts (a, h, lse, s) through an mbarrier.
//    Meanwhile the consumers already run phase 1 of the next row (up to 3
//    chunks of look-ahead), so the epilogue is off their path.
//  * Phase 2 reads the resident chunks back from TMEM (tcgen05.ld) and writes
//    dz = p (s + h((z - lse) + H)) - s[v = y] with 128-bit streaming stores.
//  * Persistent grid: one CTA per SM (18 warps), as many clusters as can be
//    co-resident, striding over rows.
//  * kA (anchor KL, regularizer_g): the anchor row's chunks ride the ring
//    beside the logits' (a z + za half-chunk pair per ring / TMEM slot), and the
//    epilogue adds KL(p || q) -- 6V bytes per row instead of the two-pass 10V.
//    kA = 3 (split stash): slices larger than TMEM keep part of the pairs in
//    shared-memory stash slots (8 TMEM + 5 shared positions per period), so a
//    Qwen-vocabulary bf16 row runs on 2-CTA clusters over all 148 SMs.
//  * Route 4 (TG_FLAG_UNSCALED_GRAD): unit row coefficients, dz = p - e_y for
//    the sequence-coupled losses; the per-row scale comes afterwards.
//  * k_fwd_tma (below) is the forward-only sibling: same ring and phase 1,
//    chunks released after phase 1, no resident rows, no cluster.
#include "tg_common.cuh"
#include "tg_rowcoef.cuh"
#include "tg_vecmath.cuh"

#include <mutex>
#include <type_traits>

namespace tg {

// Geometry (overridable at build time for A/B studies):
//   TG_CONSUMER_WARPS consumer warps + 1 epilogue warp + 1 producer warp,
//   TG_VEC_PER_THREAD 16-byte vectors per consumer thread per chunk,
//   TG_SLOTS ring slots of one chunk each (<= 227 KB of opt-in SMEM).
// Measured on B200 (V = 151,936, CL = 2): 16 x 4 x 7 (32 KB chunks, 4 consumer
// warps on every SM sub-partition) beats 14 x 4 x 8 by ~1.5 %; more warps with
// fewer vectors each, or smaller chunks, lose (scripts/gpu_libab.sh).
#ifndef TG_CONSUMER_WARPS
#define TG_CONSUMER_WARPS 16
#endif
#ifndef TG_VEC_PER_THREAD
#define TG_VEC_PER_THREAD 4
#endif
#ifndef TG_SLOTS
#define TG_SLOTS 7
#endif
constexpr int kConsumerWarps = TG_CONSUMER_WARPS;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kEpilogueWarp = kConsumerWarps;  // SM sub-partition 0
constexpr int kProducerWarp = kConsumerWarps + 1;  // sub-partition 1 (both on 0: -0.8 %)
constexpr int kFusedThreads = (kProducerWarp + 1) * 32;
constexpr int kVecPerThread = TG_VEC_PER_THREAD;  // 16-byte vectors per consumer thread per chunk
constexpr int kVecPerChunk = kConsumers * kVecPerThread;
constexpr int kChunk = kVecPerChunk * 16;         // bytes per TMA bulk copy / ring slot
constexpr int kSlots = TG_SLOTS;
static_assert(kConsumerWarps <= 32, "one partial per epilogue lane");
constexpr int kMaxPrefixChunks = 8;  // next-row phase-1 chunks run before this row's phase 2
constexpr uint32_t kPrefetchPiece = 65536;  // bytes per L2 prefetch instruction

constexpr int kMaxRingSlots = kSlots;

struct FusedSmemTail {
  uint64_t full[kMaxRingSlots];
  uint64_t empty[kMaxRingSlots];
  uint64_t pbar[2];   // consumers -> epilogue warp: per-warp partials written
  uint64_t bbar[2];   // epilogue warp -> consumers: (a, h, lse, s) written
  float4 wpart[2][4 * kConsumerWarps];  // [rank * warps + warp]: every CTA's partials
  float4 bcast[2];  // (a, h, lse, s) of a row, from the epilogue warp
  float wpart_q[2][4 * kConsumerWarps];  // kA: every CTA's anchor log-sum-exp partials
  float bcast_ca[2];                     // kA: the row's anchor coefficient ca
  float zy[2];  // CL > 1: the row's target logit, from the CTA whose slice holds it
  uint32_t tmem_base;  // TG_TMEM_STASH: 512 TMEM columns of this CTA
#ifdef TG_FUSED_PROF
  unsigned long long prof[16];
  unsigned long long post_first[2], post_last[2];
#endif
  uint64_t tfull[8];   // anchor mode 3: TMEM position filled (tcgen05.cp complete)
  uint64_t tempty[8];  // anchor mode 3: TMEM position read by phase 2 (every consumer warp)
};

// the ring + tail must fit the 227 KB per-CTA opt-in shared memory of sm_100
static_assert(size_t(kSlots) * kChunk + sizeof(FusedSmemTail) <= 232448,
              "fused kernel shared memory exceeds 227 KB");

// ---- optional cycle accounting (profiling build only: -DTG_FUSED_PROF) -------
// prof[0] consumer cycles waiting for ring data (summed over consumer warps)
// prof[1] consumer cycles waiting for the epilogue broadcast (summed over warps)
// prof[2] consumer busy span (warp 0: first wait -> last store)
// prof[3] producer cycles waiting for a free slot
// prof[4] epilogue cycles waiting for the consumer partials
// prof[5] epilogue cycles waiting for the cluster exchange
// prof[6] rows processed by the CTA
// prof[7] epilogue critical path: partials complete -> broadcast
// prof[8] epilogue: cluster exchange complete -> broadcast
// prof[9] first local warp partial posted -> epilogue wakes (all partials in)
// prof[10] first -> last local warp partial posted (intra-CTA skew)
// prof[11] / [12] anchor mode 3: consumer data waits on TMEM / shared positions
// prof[13] / [14] anchor mode 3 copier: waits for a free TMEM position / landed data
// prof[15] phase-1 chunks that took the checked path (counted per warp)
#ifdef TG_FUSED_PROF
__device__ unsigned long long g_fused_prof[1024][16];
__device__ __forceinline__ FusedSmemTail* prof_tail() {
  extern __shared__ __align__(1024) unsigned char smem[];
  return reinterpret_cast<FusedSmemTail*>(smem + size_t(kSlots) * kChunk);
}
#define TG_PROF_T0() const long long _tp0 = clock64()
#define TG_PROF_ADD(tail, i)                                                     \
  do {                                                                           \
    if ((threadIdx.x & 31) == 0)                                                 \
      atomicAdd(&(tail)->prof[i], (unsigned long long)(clock64() - _tp0));       \
  } while (0)
#else
#define TG_PROF_T0() (void)0
#define TG_PROF_ADD(tail, i) (void)0
#endif

// ---- shared-memory / barrier primitives on 32-bit shared addresses ----------

// volatile: stays ordered after the (volatile) mbarrier wait that publishes the data
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

// TG_WAIT_FULL_SLEEP: the consumers' data waits park the warp in the mbarrier
// (try_wait with a suspend-time hint) instead of re-polling (A/B; measured
// neutral for the headline, -0.4 % for 2-chunk rows: re-poll by default)
#ifndef TG_WAIT_FULL_SLEEP
#define TG_WAIT_FULL_SLEEP 0
#endif
__device__ __forceinline__ void wait_full(uint32_t bar, uint32_t parity) {
  if (TG_WAIT_FULL_SLEEP) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
  } else {
    while (!mbar_try_wait(bar, parity)) {
    }
  }
}

__device__ __forceinline__ void arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

struct RingBase {
  uint32_t ring, full, empty;  // shared addresses of slot 0's data / full / empty barrier
  uint32_t tmem;               // TMEM stash of this thread (lane, warp's column block), or 0
  uint32_t tfull;              // anchor mode 3: tfull[0] (tempty[0] follows 64 bytes later)
};

// ---- TMEM stash of the row slice (TG_TMEM_STASH) ------------------------------
// Phase 1 copies each thread's raw chunk data (kVecPerThread x 16 B = 16 fp32
// columns) into its own TMEM lane and frees the shared-memory slot at once; phase
// 2 reads it back with tcgen05.ld.  The 224 KB ring then only streams (whole-ring
// read-ahead) and the resident row slices live in the otherwise idle 256 KB of
// TMEM: warp w owns lanes 32 (w % 4) .. + 31 and columns 128 (w / 4) .. + 127,
// i.e. a ring of kTSlots chunks per warp (one 152 KB slice + a 3-chunk prefix
// of the next row at V = 151,936, CL = 2).
#ifndef TG_TMEM_STASH
#define TG_TMEM_STASH 1
#endif
constexpr bool kStash = TG_TMEM_STASH != 0;
constexpr int kTSlots = 8;
constexpr int kTCols = kVecPerThread * 4;  // 32-bit TMEM columns per thread per chunk
static_assert(!kStash || (kConsumerWarps == 16 && kTSlots * kTCols == 128),
              "stash layout: 16 consumer warps, 128 columns per warp");

__device__ __forceinline__ uint32_t stash_addr(const RingBase& rb, uint32_t chunk) {
  return rb.tmem + (chunk % uint32_t(kTSlots)) * uint32_t(kTCols);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint4 (&u)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(u[0].x), "r"(u[0].y), "r"(u[0].z), "r"(u[0].w), "r"(u[1].x), "r"(u[1].y), "r"(u[1].z),
      "r"(u[1].w), "r"(u[2].x), "r"(u[2].y), "r"(u[2].z), "r"(u[2].w), "r"(u[3].x), "r"(u[3].y),
      "r"(u[3].z), "r"(u[3].w)
      : "memory");
}

// tcgen05.cp of a [128 rows x 16 B] shared-memory matrix (rows 16 B apart: the
// no-swizzle canonical layout, 8-row core matrices 128 B apart = SBO) into 4
// TMEM columns of lanes 0..127 (row i -> lane i)
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(128u >> 4) << 16;  // leading byte offset (one core matrix wide: unused)
  d |= uint64_t(128u >> 4) << 32;  // stride byte offset: next 8 rows
  d |= uint64_t(1u) << 46;         // descriptor version (sm_100); layout 0 = no swizzle
  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}

// arrive on a CTA mbarrier once this thread's prior tcgen05 operations completed
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

// anchor mode 2: a z-only stash slot (2 vectors = 8 columns per thread), 16 per warp
constexpr int kTSlotsZ = 16;
__device__ __forceinline__ uint32_t stash_addr_z(const RingBase& rb, uint32_t chunk) {
  return rb.tmem + (chunk % uint32_t(kTSlotsZ)) * 8u;
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4& a, const uint4& b) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint4& a, uint4& b) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#ifndef TG_ZA_EVICT_LAST
#define TG_ZA_EVICT_LAST 1
#endif
__device__ __forceinline__ uint64_t policy_za() {
  uint64_t p;
  if (TG_ZA_EVICT_LAST)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// L2-resident re-read of the anchor row (mode 2): read-only path, no L1
// allocation, evict-first once consumed
__device__ __forceinline__ uint4 ld_l2_hint(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint4 (&u)[4]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(u[0].x), "=r"(u[0].y), "=r"(u[0].z), "=r"(u[0].w), "=r"(u[1].x), "=r"(u[1].y),
        "=r"(u[1].z), "=r"(u[1].w), "=r"(u[2].x), "=r"(u[2].y), "=r"(u[2].z), "=r"(u[2].w),
        "=r"(u[3].x), "=r"(u[3].y), "=r"(u[3].z), "=r"(u[3].w)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Ring position as a running chunk counter: slot = c mod kSlots, mbarrier phase
// parity = (c / kSlots) & 1 (compile-time divisor: a multiply-shift at most).
template <int NS, uint32_t CB>
struct RingItT {
  uint32_t c;
  __device__ __forceinline__ uint32_t slot() const { return c % uint32_t(NS); }
  __device__ __forceinline__ uint32_t phase() const { return (c / uint32_t(NS)) & 1u; }
  __device__ __forceinline__ uint32_t addr(const RingBase& rb) const { return rb.ring + slot() * CB; }
  __device__ __forceinline__ uint32_t full(const RingBase& rb) const { return rb.full + slot() * 8u; }
  __device__ __forceinline__ uint32_t empty(const RingBase& rb) const { return rb.empty + slot() * 8u; }
  __device__ __forceinline__ void next() { ++c; }
  __device__ __forceinline__ void advance(int n) { c += uint32_t(n); }
};
using RingIt = RingItT<kSlots, uint32_t(kChunk)>;

__device__ __forceinline__ void prefetch_l2(const char* p, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += kPrefetchPiece) {
    const uint32_t n = min(kPrefetchPiece, bytes - off);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(n) : "memory");
  }
}

// Per-CTA slice geometry (vectors of 16 bytes).
struct Slice {
  int v0, v1, nchunk, tail_vec, tail_valid;
};

// Row metadata built on the fly from the per-sequence arrays of the group
// prologue (no packed RowMeta pass): a CTA's rows ascend, so its sequence
// cursor only moves forward (amortised O(1) per row).
__device__ __forceinline__ RowMeta row_meta(const KParams& P, int64_t row, int& seq) {
  while (seq + 1 < P.n_seqs && int64_t(P.seq_off[seq + 1]) <= row) ++seq;
  RowMeta m;
  m.y = P.target[row];
  m.seq = seq;
  m.A = P.sA[seq];
  m.w = P.sW[seq];
  m.old = P.old_lp ? P.old_lp[row] : 0.f;
  m.ref = P.ref_lp ? P.ref_lp[row] : 0.f;
  if (P.pg == TG_PG_GIVEN) {  // the caller's per-row coefficient / loss (see k_rowmeta)
    m.A = P.pg_coef[row];
    m.old = P.pg_loss[row];
  }
  const bool rl = P.seq_kind == nullptr || P.seq_kind[seq] == 0;
  const bool bad = m.y < 0 || int64_t(m.y) >= P.vocab;
  m.flags = (rl ? 1u : 0u) | (bad ? 2u : 0u);
  m.ca = P.anchor_beta > 0.f ? P.anchor_beta / P.sK[seq] : 0.f;
  return m;
}

// first sequence containing `row` (binary search over the prefix sums)
__device__ __forceinline__ int seq_of_row(const KParams& P, int64_t row) {
  int lo = 0, hi = P.n_seqs;  // invariant: seq_off[lo] <= row < seq_off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (int64_t(P.seq_off[mid]) <= row) lo = mid; else hi = mid;
  }
  return lo;
}

// ---- phase 1: one chunk (kVecPerThread vectors per consumer thread) ---------
#ifndef TG_SKIP_EMPTY
#define TG_SKIP_EMPTY 1
#endif
// kPartial: the chunk may run past the slice end (lanes there load a neutral
// -1e30 vector, which adds exactly 0 to the sums, so every lane takes part in
// the warp vote).  kMaskTail: the chunk holds the tail padding.
//
// Speculative fast path: the sums are taken straight away with the current
// reference max m (warp-uniform under kWM) -- no -inf clamp, no vector max, no
// pre-vote -- and accepted when they are safe: finite, s <= 2^32 (no term near
// overflow) and, for the first chunk of a row (m carried over from the
// previous row), s >= 2^-20 (no significant term lost to underflow).  Otherwise
// (a -inf logit gives 0 * -inf = NaN in the sum of p z, a new maximum more
// than ~22 above m, the first rows) the warp redoes the chunk on the checked
// path: clamp, vector max, rescale, sums.  Partial and tail chunks take the
// same speculative path (neutral / masked elements contribute exactly 0).
struct Acc1 {
  Acc2 a;
  bool fresh;  // no chunk of the current row accumulated yet (warp-uniform)
};

// kWM: the reference max m is warp-uniform -- the checked path takes the warp's
// maximum (one REDUX on an order-preserving integer image of the floats) -- so a
// warp's per-row partial is (m, sum s, sum t), plain butterfly sums instead of a
// 5-level online merge.  Measured: +6 % at V = 32,000 (2-chunk rows), +0.4 % at
// V = 151,936 (3 % fewer cycles per row in the instrumented build).
__device__ __forceinline__ float warp_max_f(float v) {
  const int i = __float_as_int(v);
  const int key = __reduce_max_sync(0xffffffffu, i >= 0 ? i : i ^ 0x7fffffff);
  return __int_as_float(key >= 0 ? key : key ^ 0x7fffffff);
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// the warp's partial of the current row (neutral when the warp saw nothing);
// kWM: m is warp-uniform, plain sums; otherwise an online merge of lane partials
template <bool kWM>
__device__ __forceinline__ Online warp_partial(const Acc1& acc) {
  float s0, s1, t0, t1;
  upk2(acc.a.s2, s0, s1);
  upk2(acc.a.t2, t0, t1);
  float s = s0 + s1, t = t0 + t1;
  if constexpr (kWM) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, d);
      t += __shfl_xor_sync(0xffffffffu, t, d);
    }
    return Online{s > 0.f ? acc.a.m : kNegInf, s, t};
  } else {
    // a lane that saw no element of the row carries a stale m: neutral
    return warp_merge(Online{s > 0.f ? acc.a.m : kNegInf, s, t});
  }
}

template <typename T, bool kPartial, bool kMaskTail, bool kWM>
__device__ __forceinline__ void phase1_checked(Acc1& acc, uint4 (&u)[kVecPerThread],
                                               const bool (&valid)[kVecPerThread], int vbase,
                                               const Slice& sl, int tid) {
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    Pk<T>::clamp(u[g]);
    if (kMaskTail && vec == sl.tail_vec) Pk<T>::mask_from(u[g], sl.tail_valid);
  }
  const float gmax = group_max<T>(u);
  const float vmax = kWM ? warp_max_f(gmax) : gmax;
  if (acc.fresh) {  // empty sums: take this chunk's (warp) max as the reference
    acc.a.m = vmax;
    const float nmL = -vmax * kLog2e;
    acc.a.nm2 = pk2(nmL, nmL);
  } else {
    rescale(acc.a, vmax);
  }
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g)
    if (!kPartial || valid[g]) accumulate<T>(acc.a, u[g]);
  acc.fresh = false;
}

template <typename T, bool kPartial, bool kMaskTail, bool kStashRow = false, bool kWM = false>
__device__ __forceinline__ void phase1_chunk(Acc1& acc, RingIt& it, const RingBase& rb,
                                             int vbase, const Slice& sl, int tid) {
  uint4 u[kVecPerThread];
  bool valid[kVecPerThread];
  {
    TG_PROF_T0();
    wait_full(it.full(rb), it.phase());
    TG_PROF_ADD(prof_tail(), 0);
  }
  const uint32_t a = it.addr(rb) + tid * 16;
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    valid[g] = !kPartial || vec < sl.v1;
    u[g] = valid[g] ? lds128(a + g * kConsumers * 16) : Pk<T>::neutral();
  }
  if constexpr (kStashRow) {
    static_assert(kVecPerThread == 4, "16-column stash");
    tmem_st16(stash_addr(rb, it.c), u);  // raw data, for phase 2
    __syncwarp();
    if ((tid & 31) == 0) arrive_u32(it.empty(rb));  // the slot streams on
  }
  it.next();
  {
    // partial chunks: lanes past the slice hold the neutral -1e30 vector (p = 0,
    // p z = 0); the tail vector's columns >= V are masked to -1e30 the same way
    if constexpr (kMaskTail) {
#pragma unroll
      for (int g = 0; g < kVecPerThread; ++g)
        if (vbase + g * kConsumers + tid == sl.tail_vec) Pk<T>::mask_from(u[g], sl.tail_valid);
    }
    const uint64_t l2e2 = pk2(kLog2e, kLog2e);
    uint64_t s2 = pk2(0.f, 0.f), t2 = pk2(0.f, 0.f);
#pragma unroll
    for (int g = 0; g < kVecPerThread; ++g) {
      // a vector past the slice end for the whole (virtual) warp adds exactly
      // 0: skip its math (the last, partial chunk of a slice)
      if (kPartial && TG_SKIP_EMPTY && vbase + g * kConsumers + (tid & ~31) >= sl.v1) continue;
#pragma unroll
      for (int w = 0; w < Vec<T>::N / 2; ++w) {
        const uint64_t x = pair<T>(u[g], w);
        const uint64_t p = ex2x2(fma2(x, l2e2, acc.a.nm2));
        s2 = add2(s2, p);
        t2 = fma2(p, x, t2);
      }
    }
    float s0, s1, t0, t1;
    upk2(s2, s0, s1);
    upk2(t2, t0, t1);
    const float sc = s0 + s1, tc = t0 + t1;
    bool ok;
    if constexpr (kWM) {
      ok = __all_sync(0xffffffffu, sc <= 4294967296.0f && fabsf(tc) <= 3.0e38f);
      if (ok && acc.fresh)  // stale m from the previous row: the warp must keep 2^-20
        ok = warp_sum_f(sc) >= 9.5367431640625e-07f;
    } else {
      ok = __all_sync(0xffffffffu, sc <= 4294967296.0f && fabsf(tc) <= 3.0e38f &&
                                       (!acc.fresh || sc >= 9.5367431640625e-07f));
    }
    if (ok) {
      acc.a.s2 = add2(acc.a.s2, s2);
      acc.a.t2 = add2(acc.a.t2, t2);
      acc.fresh = false;
      return;
    }
  }
#ifdef TG_FUSED_PROF
  if ((tid & 31) == 0) atomicAdd(&prof_tail()->prof[15], 1ull);  // checked-path chunks (warps)
#endif
  phase1_checked<T, kPartial, kMaskTail, kWM>(acc, u, valid, vbase, sl, tid);
}

// ---- phase 2: dz for one chunk ------------------------------------------------
template <typename T, bool kHasH, bool kCheck>
__device__ __forceinline__ void phase2_chunk(const RingIt& it, const RingBase& rb, int vbase,
                                             const Slice& sl, char* dzrow, int vy, int ye,
                                             float s_t, uint64_t nl2, uint64_t av2, uint64_t hz2,
                                             int tid) {
  constexpr int EPV = Vec<T>::N;
  char* dst = dzrow + int64_t(vbase + tid) * 16;
  const uint32_t a = it.addr(rb) + tid * 16;
  uint4 su[kVecPerThread];
  if constexpr (kStash) tmem_ld16(stash_addr(rb, it.c), su);  // whole warp, before any branch
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    if (!kCheck || vec < sl.v1) {
      float d[EPV];
      dz_vec<T, kHasH>(kStash ? su[g] : lds128(a + g * kConsumers * 16), d, nl2, av2, hz2);
      bool done = false;
      if (kCheck) {
        if (vec == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e == ye) d[e] -= s_t;
        }
        if (vec == sl.tail_vec) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e < sl.tail_valid) Vec<T>::store1(dzrow, int64_t(vec) * EPV + e, d[e]);
          done = true;
        }
      }
#ifdef TG_NULL_MATH
      if (!done) st_stream(dst + g * kConsumers * 16, lds128(a + g * kConsumers * 16));
#else
      if (!done) st_stream(dst + g * kConsumers * 16, Vec<T>::pack(d));
#endif
    }
  }
}

// phase 2 over one row; the chunk holding the target logit or tail padding, and
// the last partial chunk, take the checked variant.
template <typename T, bool kHasH>
__device__ __forceinline__ void phase2_row(const Slice& sl, RingIt it, const RingBase& rb,
                                           char* dzrow, int vy, int ye, float s_t, uint64_t nl2,
                                           uint64_t av2, uint64_t hz2, int tid, int lane) {
  int vbase = sl.v0;
  for (int j = 0; j < sl.nchunk; ++j) {
    const int vend = vbase + kVecPerChunk;
    const bool check = (vend > sl.v1) || (sl.tail_vec >= vbase && sl.tail_vec < vend) ||
                       (vy >= vbase && vy < vend);
    if (check)
      phase2_chunk<T, kHasH, true>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2,
                                               tid);
    else
      phase2_chunk<T, kHasH, false>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2,
                                                tid);
    if constexpr (!kStash) {  // (stash: the slot was freed in phase 1)
      __syncwarp();
      if (lane == 0) arrive_u32(it.empty(rb));
    }
    it.next();
    vbase = vend;
  }
}

// phase 1 over chunks [c0, c1) of a row whose first chunk is at `row_it`
template <typename T, bool kWM>
__device__ __forceinline__ void phase1_range(Acc1& acc, RingIt row_it, const RingBase& rb,
                                             const Slice& sl, int c0, int c1, int tid) {
  RingIt it = row_it;
  it.advance(c0);
  int vbase = sl.v0 + c0 * kVecPerChunk;
  for (int c = c0; c < c1; ++c) {
    const int vend = vbase + kVecPerChunk;
    const bool has_tail = sl.tail_vec >= vbase && sl.tail_vec < vend;
    if (vend <= sl.v1 && !has_tail)
      phase1_chunk<T, false, false, kStash, kWM>(acc, it, rb, vbase, sl, tid);
    else if (!has_tail)
      phase1_chunk<T, true, false, kStash, kWM>(acc, it, rb, vbase, sl, tid);
    else
      phase1_chunk<T, true, true, kStash, kWM>(acc, it, rb, vbase, sl, tid);
    vbase = vend;
  }
}

// new row: empty sums; the reference max carries over from the previous row
// (the fast path's bet that consecutive rows have similar maxima)
__device__ __forceinline__ void acc_new_row(Acc1& acc) {
  acc.a.s2 = pk2(0.f, 0.f);
  acc.a.t2 = pk2(0.f, 0.f);
  acc.fresh = true;
}

__device__ __forceinline__ Acc1 acc_init() {
  Acc1 acc;
  acc.a.m = 0.f;
  acc.a.nm2 = pk2(0.f, 0.f);
  acc_new_row(acc);
  return acc;
}

// ---- the epilogue's merge of the CL x warps row partials ----------------------
// REDUX form: one warp max of the partials' reference maxima, each partial
// scaled once, then plain butterfly sums -- a short dependency chain instead of
// log2(NP) levels of online merges.  Measured: +10.5 % for the fused anchor
// path at CL = 4 (64 partials, three merges: critical path 5.1k -> 3.9k cycles
// per row), but -0.4 % (headline, CL = 2) and -2.3 % (CL = 1) for one merge of
// <= 32 partials, so it is used only for the former.
#ifndef TG_MERGE_REDUX
#define TG_MERGE_REDUX 1
#endif
template <int NP, bool kU>
__device__ __forceinline__ float4 merge_partials(const float4* wp, int lane) {
  constexpr int K = (NP + 31) / 32;
  float4 v[K];
  float mloc = kNegInf;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < NP ? wp[j] : make_float4(kNegInf, 0.f, 0.f, 0.f);
    mloc = fmaxf(mloc, v[i].x);
  }
  const float M = warp_max_f(mloc);
  float S = 0.f, Tt = 0.f, U = 0.f;
  if (M != kNegInf) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const float f = v[i].x == kNegInf ? 0.f : ex2((v[i].x - M) * kLog2e);
      S = fmaf(v[i].y, f, S);
      Tt = fmaf(v[i].z, f, Tt);
      if (kU) U = fmaf(v[i].w, f, U);
    }
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    S += __shfl_xor_sync(0xffffffffu, S, d);
    Tt += __shfl_xor_sync(0xffffffffu, Tt, d);
    if (kU) U += __shfl_xor_sync(0xffffffffu, U, d);
  }
  return make_float4(M, S, Tt, U);
}

// the previous form: online merges (kept for A/B: -DTG_MERGE_REDUX=0)
template <int NP, bool kU>
__device__ __forceinline__ float4 merge_partials_online(const float4* wp, int lane) {
  Online a = {kNegInf, 0.f, 0.f}, b = {kNegInf, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < (NP + 31) / 32; ++i) {
    const int j = lane + 32 * i;
    if (j < NP) {
      const float4 v = wp[j];
      a = online_merge(a, Online{v.x, v.y, v.z});
      if (kU) b = online_merge(b, Online{v.x, v.y, v.w});
    }
  }
  a = warp_merge_first<(NP < 32 ? NP : 32)>(a);
  if (kU) b = warp_merge_first<(NP < 32 ? NP : 32)>(b);
  return make_float4(a.m, a.s, a.t, b.t);
}

// log-sum-exp of NP per-warp log-sum-exps by online merges (lane 0 gets it)
template <int NP>
__device__ __forceinline__ float merge_lse_online(const float* lq, int lane) {
  Online q = {kNegInf, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < (NP + 31) / 32; ++i) {
    const int j = lane + 32 * i;
    if (j < NP) q = online_merge(q, Online{lq[j], lq[j] > kNegInf ? 1.f : 0.f, 0.f});
  }
  q = warp_merge_first<(NP < 32 ? NP : 32)>(q);
  return q.m + logf(q.s);
}

// log-sum-exp of NP per-warp log-sum-exps (all lanes get it)
template <int NP>
__device__ __forceinline__ float merge_lse(const float* lq, int lane) {
  constexpr int K = (NP + 31) / 32;
  float v[K];
  float mloc = kNegInf;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < NP ? lq[j] : kNegInf;
    mloc = fmaxf(mloc, v[i]);
  }
  const float M = warp_max_f(mloc);
  if (M == kNegInf) return kNegInf;
  float S = 0.f;
#pragma unroll
  for (int i = 0; i < K; ++i) S += v[i] == kNegInf ? 0.f : ex2((v[i] - M) * kLog2e);
  return M + logf(warp_sum_f(S));
}

// ---- fused anchor KL (regularizer_g, algorithms.py:193-217) -------------------
// kA: the row's anchor logits za ride the same ring -- every ring slot holds a
// half chunk of z (kVA vectors per consumer thread) followed by the za half
// chunk of the same columns, and one TMEM stash slot keeps both -- so each
// row costs 6V bytes (z and za read once, dz written once) instead of the
// two-pass route's 10V, with the same look-ahead in columns as the default
// path.
// Phase 1 adds Sigma p (z - za) (aligned with z's reference max) and the
// anchor's own online sum; the epilogue forms lse_q and KL(p || q); phase 2
// writes dz = p (a + hz z - ca za) - s [v = y] (k_bwd's formula).
//
// Slot geometry per anchor mode (kA):
//   1: 32 KB ring slots (2 z + 2 za vectors per thread), one 16-column TMEM slot
//      per ring slot (8 per warp);
//   2: the same ring, z only in 8-column TMEM slots (16 per warp), za re-read
//      from L2 in phase 2.
// (Measured and dropped, profiles/r02_anchor_modes.txt: 16 KB ring slots with
// z + za in 8-column TMEM slots -- 13 slots per 3-CTA slice leave 3 of look-
// ahead -- ran 10-18 % slower than mode 1: the per-slot costs double.)
//   3: split stash -- the row slices are larger than TMEM (a 2-CTA slice at
//      V = 151,936 bf16 is 10 z + za pairs = 304 KB), so the stash is a ring of
//      kTSlots + kSSlots positions: positions 0..7 of every period are TMEM
//      slots (the pair lands in one of kLSlots shared-memory landing slots and
//      phase 1 copies it to TMEM, as in mode 1), positions 8.. are shared-memory
//      stash slots (the pair lands there and stays until phase 2 has read it
//      again).  TMEM 256 KB + 5 x 32 KB shared = 13 pairs resident: a 10-pair
//      slice + 3 of look-ahead, on all 148 SMs (2-CTA clusters) instead of the
//      132 that 4-CTA clusters of mode 1 occupy.
constexpr int kVA = kVecPerThread / 2;  // z (and za) vectors per thread per slot

#ifndef TG_ANCHOR_SSLOTS
#define TG_ANCHOR_SSLOTS 5
#endif
constexpr int kSSlots = TG_ANCHOR_SSLOTS;   // mode 3: shared-memory stash slots
// Mode 3, TMEM positions: by default the consumers copy each landed pair into
// TMEM in phase 1 (lds + tcgen05.st, as mode 1) and free the landing slot; the
// producer keeps the pairs behind the landing slots in L2 (bulk prefetch a few
// positions ahead, TG_PREFETCH_CHUNKS).  TG_SPLIT_UTCCP=1 (A/B build variant):
// a copier lane moves each landed pair into TMEM with tcgen05.cp (4 column
// blocks x 4 vectors of 128 lanes x 16 B) once the TMEM position is free and
// frees the landing slot on the copy's commit -- parity-green, but 4.90 vs
// 5.21 TB/s (profiles/r02_anchor_split.txt): the copier shares the producer
// warp's issue with the two TMA lanes, and the consumers then wait on the
// copies (18 % of the span on TMEM positions).
#ifndef TG_SPLIT_UTCCP
#define TG_SPLIT_UTCCP 0
#endif
constexpr bool kSplitCp = TG_SPLIT_UTCCP != 0;
// Sanitizer study (-DTG_ARRIVE_ALL): every consumer thread arrives on the mode-3
// slot barriers, and every epilogue lane on the broadcast barrier, instead of
// one lane per warp after __syncwarp / the warp's shuffles -- racecheck does not
// follow that release chain (profiles/r02_sanitizer.txt)
#ifndef TG_ARRIVE_ALL
#define TG_ARRIVE_ALL 0
#endif
constexpr bool kArriveAll = TG_ARRIVE_ALL != 0;
constexpr int kLSlots = kSlots - kSSlots;   // mode 3: landing slots of the TMEM positions
static_assert(kSSlots >= 1 && kLSlots >= 1, "mode 3 needs stash and landing slots");
static_assert(kTSlots == 8, "FusedSmemTail::tfull / tempty hold one barrier per TMEM position");

// Mode-3 stash position as a running counter c (same protocol as RingItT):
// period kP = kTSlots + kSSlots; pos = c mod kP.  TMEM position (pos < kTSlots):
// landing slot = (t mod kLSlots), t = the running count of TMEM positions, its
// mbarrier phase (t / kLSlots) & 1; shared stash position: slot kLSlots + pos -
// kTSlots, phase (c / kP) & 1.  Buffer / barrier index = the slot.
template <uint32_t CB>
struct SplitItT {
  static constexpr uint32_t kP = uint32_t(kTSlots + kSSlots);
  uint32_t c;
  __device__ __forceinline__ uint32_t pos() const { return c % kP; }
  __device__ __forceinline__ bool in_tmem() const { return pos() < uint32_t(kTSlots); }
  __device__ __forceinline__ uint32_t tcount() const {
    return (c / kP) * uint32_t(kTSlots) + pos();
  }
  __device__ __forceinline__ uint32_t slot() const {
    return in_tmem() ? tcount() % uint32_t(kLSlots) : uint32_t(kLSlots) + pos() - uint32_t(kTSlots);
  }
  __device__ __forceinline__ uint32_t phase() const {
    return (in_tmem() ? tcount() / uint32_t(kLSlots) : c / kP) & 1u;
  }
  __device__ __forceinline__ uint32_t addr(const RingBase& rb) const { return rb.ring + slot() * CB; }
  __device__ __forceinline__ uint32_t full(const RingBase& rb) const { return rb.full + slot() * 8u; }
  __device__ __forceinline__ uint32_t empty(const RingBase& rb) const { return rb.empty + slot() * 8u; }
  __device__ __forceinline__ uint32_t tmem(const RingBase& rb) const {
    return rb.tmem + pos() * uint32_t(kTCols);
  }
  // TMEM position barriers (tcgen05.cp landing) and their phase
  __device__ __forceinline__ uint32_t tfull(const RingBase& rb) const { return rb.tfull + pos() * 8u; }
  __device__ __forceinline__ uint32_t tempty(const RingBase& rb) const {
    return rb.tfull + 64u + pos() * 8u;
  }
  __device__ __forceinline__ uint32_t tphase() const { return (c / kP) & 1u; }
  __device__ __forceinline__ void next() { ++c; }
  __device__ __forceinline__ void advance(int n) { c += uint32_t(n); }
};

template <int M>
struct AGeo {
  static constexpr int VA = kVA;                           // z vectors per thread per slot
  static constexpr int VPC = kConsumers * VA;              // z vectors per slot
  static constexpr uint32_t HALF = uint32_t(VPC) * 16u;    // bytes of z (= of za) per slot
  static constexpr int SLOTS = kSlots;
  static constexpr uint32_t CHUNK = 2u * HALF;             // ring slot bytes
  // resident positions per warp (the stash ring's period)
  static constexpr int TSLOTS = (M == 1) ? kTSlots : (M == 2) ? kTSlotsZ : kTSlots + kSSlots;
  using It = typename std::conditional<M == 3, SplitItT<CHUNK>, RingItT<SLOTS, CHUNK>>::type;
};
static_assert(AGeo<1>::CHUNK == uint32_t(kChunk), "a z + za slot is one ring slot");

struct AccA {
  Acc1 z;         // (m, nm2, s2, t2, fresh) of the logits
  uint64_t u2;    // Sigma p (z - za), p = 2^((z - m) log2e)
  float mq;       // anchor reference max (warp-uniform)
  uint64_t nmq2;  // (-mq log2e, -mq log2e)
  uint64_t sq2;   // Sigma 2^((za - mq) log2e)
};

__device__ __forceinline__ void acc_new_row_a(AccA& acc) {
  acc.z.a.s2 = pk2(0.f, 0.f);
  acc.z.a.t2 = pk2(0.f, 0.f);
  acc.z.fresh = true;
  acc.u2 = pk2(0.f, 0.f);
  acc.sq2 = pk2(0.f, 0.f);
}

__device__ __forceinline__ AccA acc_init_a() {
  AccA acc;
  acc.z.a.m = 0.f;
  acc.z.a.nm2 = pk2(0.f, 0.f);
  acc.mq = 0.f;
  acc.nmq2 = pk2(0.f, 0.f);
  acc_new_row_a(acc);
  return acc;
}

// z, za pairs of one vector pair: the sums of one chunk
template <typename T>
__device__ __forceinline__ void accumulate_a(const uint4& uz, const uint4& uq, uint64_t nm2,
                                             uint64_t nmq2, uint64_t& s2, uint64_t& t2,
                                             uint64_t& u2, uint64_t& sq2) {
  const uint64_t l2e2 = pk2(kLog2e, kLog2e), neg2 = pk2(-1.f, -1.f);
#pragma unroll
  for (int w = 0; w < Vec<T>::N / 2; ++w) {
    const uint64_t x = pair<T>(uz, w), xq = pair<T>(uq, w);
    const uint64_t p = ex2x2(fma2(x, l2e2, nm2));
    s2 = add2(s2, p);
    t2 = fma2(p, x, t2);
    u2 = fma2(p, fma2(xq, neg2, x), u2);
    sq2 = add2(sq2, ex2x2(fma2(xq, l2e2, nmq2)));
  }
}

template <typename T, int kMode, bool kPartial, bool kMaskTail>
__device__ __forceinline__ void phase1_chunk_a(AccA& acc, typename AGeo<kMode>::It& it,
                                               const RingBase& rb, int vbase, const Slice& sl,
                                               int tid) {
  constexpr int kVA = AGeo<kMode>::VA;
  constexpr uint32_t kHalf = AGeo<kMode>::HALF;
  uint4 u[2 * kVA];  // [0, kVA): z vectors, [kVA, 2 kVA): za vectors of the same columns
  bool valid[kVA];
  // mode 3 with the copier: a TMEM position's pair is read from TMEM once the
  // tcgen05.cp into it completed
  bool from_tmem = false;
  if constexpr (kMode == 3 && kSplitCp) {
    from_tmem = it.in_tmem();
    TG_PROF_T0();
    if (from_tmem)
      wait_full(it.tfull(rb), it.tphase());
    else
      wait_full(it.full(rb), it.phase());
    TG_PROF_ADD(prof_tail(), 0);
#ifdef TG_FUSED_PROF
    if ((threadIdx.x & 31) == 0)
      atomicAdd(&prof_tail()->prof[from_tmem ? 11 : 12], (unsigned long long)(clock64() - _tp0));
#endif
  } else {
    TG_PROF_T0();
    wait_full(it.full(rb), it.phase());
    TG_PROF_ADD(prof_tail(), 0);
  }
  if (from_tmem) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (kMode == 3) tmem_ld16(it.tmem(rb), u);
#pragma unroll
    for (int g = 0; g < kVA; ++g) {
      valid[g] = !kPartial || vbase + g * kConsumers + tid < sl.v1;
      if (!valid[g]) {
        u[g] = Pk<T>::neutral();
        u[kVA + g] = Pk<T>::neutral();
      }
    }
  } else {
    const uint32_t a = it.addr(rb) + tid * 16;
#pragma unroll
    for (int g = 0; g < kVA; ++g) {
      const int vec = vbase + g * kConsumers + tid;
      valid[g] = !kPartial || vec < sl.v1;
      u[g] = valid[g] ? lds128(a + g * kConsumers * 16) : Pk<T>::neutral();
      u[kVA + g] = valid[g] ? lds128(a + kHalf + g * kConsumers * 16) : Pk<T>::neutral();
    }
  }
  if constexpr (kMode == 3) {  // TMEM position: copy out, free the landing slot;
    if (!kSplitCp && it.in_tmem()) {  // shared stash position: kept until phase 2
      tmem_st16(it.tmem(rb), u);
      __syncwarp();
      if (kArriveAll || (tid & 31) == 0) arrive_u32(it.empty(rb));
    }
  } else {
    if constexpr (kMode == 1)
      tmem_st16(stash_addr(rb, it.c), u);  // z, z, za, za
    else  // mode 2: z, z (za is re-read from L2 in phase 2)
      tmem_st8(stash_addr_z(rb, it.c), u[0], u[1]);
    __syncwarp();
    if ((tid & 31) == 0) arrive_u32(it.empty(rb));
  }
  it.next();
  if constexpr (kMaskTail) {
#pragma unroll
    for (int g = 0; g < kVA; ++g)
      if (vbase + g * kConsumers + tid == sl.tail_vec) {
        Pk<T>::mask_from(u[g], sl.tail_valid);
        Pk<T>::mask_from(u[kVA + g], sl.tail_valid);
      }
  }
  {  // speculative: the current reference maxima, accepted when the sums are safe
    uint64_t s2 = pk2(0.f, 0.f), t2 = s2, u2 = s2, sq2 = s2;
#pragma unroll
    for (int g = 0; g < kVA; ++g) {
      // (a vector past the slice end for the whole virtual warp adds exactly 0)
      if (kPartial && TG_SKIP_EMPTY && vbase + g * kConsumers + (tid & ~31) >= sl.v1) continue;
      accumulate_a<T>(u[g], u[kVA + g], acc.z.a.nm2, acc.nmq2, s2, t2, u2, sq2);
    }
    float a0, a1;
    upk2(s2, a0, a1);
    const float sc = a0 + a1;
    upk2(t2, a0, a1);
    const float tc = a0 + a1;
    upk2(u2, a0, a1);
    const float uc = a0 + a1;
    upk2(sq2, a0, a1);
    const float qc = a0 + a1;
    bool ok = __all_sync(0xffffffffu, sc <= 4294967296.0f && qc <= 4294967296.0f &&
                                          fabsf(tc) <= 3.0e38f && fabsf(uc) <= 3.0e38f);
    if (ok && acc.z.fresh)
      ok = warp_sum_f(sc) >= 9.5367431640625e-07f && warp_sum_f(qc) >= 9.5367431640625e-07f;
    if (ok) {
      acc.z.a.s2 = add2(acc.z.a.s2, s2);
      acc.z.a.t2 = add2(acc.z.a.t2, t2);
      acc.u2 = add2(acc.u2, u2);
      acc.sq2 = add2(acc.sq2, sq2);
      acc.z.fresh = false;
      return;
    }
  }
  // checked: clamp -inf, exact warp maxima, rescale, sums
  uint4 uz[kVA], uq[kVA];
#pragma unroll
  for (int g = 0; g < kVA; ++g) {
    uz[g] = u[g];
    uq[g] = u[kVA + g];
    Pk<T>::clamp(uz[g]);
    Pk<T>::clamp(uq[g]);
  }
  const float vmax = warp_max_f(group_max<T>(uz));
  const float qmax = warp_max_f(group_max<T>(uq));
  if (acc.z.fresh) {
    acc.z.a.m = vmax;
    acc.mq = qmax;
  } else {
    if (vmax > acc.z.a.m) {
      const float f = ex2((acc.z.a.m - vmax) * kLog2e);
      const uint64_t f2 = pk2(f, f);
      acc.z.a.s2 = mul2(acc.z.a.s2, f2);
      acc.z.a.t2 = mul2(acc.z.a.t2, f2);
      acc.u2 = mul2(acc.u2, f2);
      acc.z.a.m = vmax;
    }
    if (qmax > acc.mq) {
      const float f = ex2((acc.mq - qmax) * kLog2e);
      acc.sq2 = mul2(acc.sq2, pk2(f, f));
      acc.mq = qmax;
    }
  }
  const float nmL = -acc.z.a.m * kLog2e, nqL = -acc.mq * kLog2e;
  acc.z.a.nm2 = pk2(nmL, nmL);
  acc.nmq2 = pk2(nqL, nqL);
#pragma unroll
  for (int g = 0; g < kVA; ++g)
    if (!kPartial || valid[g])
      accumulate_a<T>(uz[g], uq[g], acc.z.a.nm2, acc.nmq2, acc.z.a.s2, acc.z.a.t2, acc.u2,
                      acc.sq2);
  acc.z.fresh = false;
}

// logical chunks [c0, c1) of a row whose first ring position is `row_it`
template <typename T, int kMode>
__device__ __forceinline__ void phase1_range_a(AccA& acc, typename AGeo<kMode>::It row_it,
                                               const RingBase& rb, const Slice& sl, int c0,
                                               int c1, int tid) {
  constexpr int kVecPerChunkA = AGeo<kMode>::VPC;
  typename AGeo<kMode>::It it = row_it;
  it.advance(c0);
  int vbase = sl.v0 + c0 * kVecPerChunkA;
  for (int c = c0; c < c1; ++c) {
    const int vend = vbase + kVecPerChunkA;
    const bool has_tail = sl.tail_vec >= vbase && sl.tail_vec < vend;
    if (vend <= sl.v1 && !has_tail)
      phase1_chunk_a<T, kMode, false, false>(acc, it, rb, vbase, sl, tid);
    else if (!has_tail)
      phase1_chunk_a<T, kMode, true, false>(acc, it, rb, vbase, sl, tid);
    else
      phase1_chunk_a<T, kMode, true, true>(acc, it, rb, vbase, sl, tid);
    vbase = vend;
  }
}

// the warp's (m, Sigma s, Sigma t, Sigma u) and the anchor's log-sum-exp
__device__ __forceinline__ float4 warp_partial_a(const AccA& acc, float& lq) {
  float s0, s1;
  upk2(acc.z.a.s2, s0, s1);
  float s = s0 + s1;
  upk2(acc.z.a.t2, s0, s1);
  float t = s0 + s1;
  upk2(acc.u2, s0, s1);
  float u = s0 + s1;
  upk2(acc.sq2, s0, s1);
  float q = s0 + s1;
  s = warp_sum_f(s);
  t = warp_sum_f(t);
  u = warp_sum_f(u);
  q = warp_sum_f(q);
  lq = q > 0.f ? acc.mq + logf(q) : kNegInf;
  return make_float4(s > 0.f ? acc.z.a.m : kNegInf, s, t, u);
}

// phase 2 of one logical chunk: z and za from the two stash slots
// (mode 2: z from the stash, za = q[] re-read from L2 by the caller)
template <typename T, int kMode, bool kCheck>
__device__ __forceinline__ void phase2_chunk_a(const typename AGeo<kMode>::It& it,
                                               const RingBase& rb, int vbase, const Slice& sl,
                                               char* dzrow, int vy, int ye, float s_t,
                                               uint64_t nl2, uint64_t av2, uint64_t hz2,
                                               uint64_t nca2, int tid,
                                               const uint4 (&q)[AGeo<kMode>::VA]) {
  constexpr int kVA = AGeo<kMode>::VA;
  constexpr int EPV = Vec<T>::N;
  char* dst = dzrow + int64_t(vbase + tid) * 16;
  uint4 su[2 * kVA];
  if constexpr (kMode == 2) {
    tmem_ld8(stash_addr_z(rb, it.c), su[0], su[1]);
#pragma unroll
    for (int g = 0; g < kVA; ++g) su[kVA + g] = q[g];
  } else if constexpr (kMode == 3) {
    if (it.in_tmem()) {
      tmem_ld16(it.tmem(rb), su);
    } else {  // the pair is still in its shared-memory stash slot
      const uint32_t a = it.addr(rb) + tid * 16;
#pragma unroll
      for (int g = 0; g < kVA; ++g) {
        su[g] = lds128(a + g * kConsumers * 16);
        su[kVA + g] = lds128(a + AGeo<kMode>::HALF + g * kConsumers * 16);
      }
    }
  } else {
    tmem_ld16(stash_addr(rb, it.c), su);
  }
  const uint64_t l2e2 = pk2(kLog2e, kLog2e);
#pragma unroll
  for (int g = 0; g < kVA; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    if (!kCheck || vec < sl.v1) {
      uint4 uz = su[g], uq = su[kVA + g];
      Pk<T>::clamp(uz);
      Pk<T>::clamp(uq);
      float d[EPV];
#pragma unroll
      for (int w = 0; w < EPV / 2; ++w) {
        const uint64_t x = pair<T>(uz, w), xq = pair<T>(uq, w);
        const uint64_t p = ex2x2(fma2(x, l2e2, nl2));
        const uint64_t c = fma2(nca2, xq, fma2(hz2, x, av2));
        upk2(mul2(p, c), d[2 * w], d[2 * w + 1]);
      }
      bool done = false;
      if (kCheck) {
        if (vec == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e == ye) d[e] -= s_t;
        }
        if (vec == sl.tail_vec) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e < sl.tail_valid) Vec<T>::store1(dzrow, int64_t(vec) * EPV + e, d[e]);
          done = true;
        }
      }
      if (!done) st_stream(dst + g * kConsumers * 16, Vec<T>::pack(d));
    }
  }
  if constexpr (kMode == 3) {  // a shared stash slot is free once every warp read it
    if (!it.in_tmem()) {
      __syncwarp();
      if (kArriveAll || (tid & 31) == 0) arrive_u32(it.empty(rb));
    } else if constexpr (kSplitCp) {  // the TMEM position, for the copier
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if ((tid & 31) == 0) arrive_u32(it.tempty(rb));
    }
  }
}

// mode 2: the za vectors of one chunk from L2 (neutral past the slice end)
template <typename T, int kVA>
__device__ __forceinline__ void load_za(uint4 (&q)[kVA], const char* qrow, int vbase,
                                        const Slice& sl, int tid, uint64_t pol) {
#pragma unroll
  for (int g = 0; g < kVA; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    q[g] = vec < sl.v1 ? ld_l2_hint(qrow + int64_t(vec) * 16, pol) : Pk<T>::neutral();
  }
}

template <typename T, int kMode>
__device__ __forceinline__ void phase2_row_a(const Slice& sl, typename AGeo<kMode>::It it,
                                             const RingBase& rb, const char* qrow, char* dzrow,
                                             int vy, int ye, float s_t, uint64_t nl2,
                                             uint64_t av2, uint64_t hz2, uint64_t nca2, int tid,
                                             uint64_t pol) {
  constexpr int kVA = AGeo<kMode>::VA;
  constexpr int kVecPerChunkA = AGeo<kMode>::VPC;
  int vbase = sl.v0;
  uint4 q[kVA];
  // mode 2: the za loads run one chunk ahead of their use (L2 latency)
  if constexpr (kMode == 2) load_za<T, kVA>(q, qrow, vbase, sl, tid, pol);
  for (int j = 0; j < sl.nchunk; ++j) {
    const int vend = vbase + kVecPerChunkA;
    uint4 qn[kVA];
    if constexpr (kMode == 2) {
      if (j + 1 < sl.nchunk) load_za<T, kVA>(qn, qrow, vend, sl, tid, pol);
    }
    const bool check = (vend > sl.v1) || (sl.tail_vec >= vbase && sl.tail_vec < vend) ||
                       (vy >= vbase && vy < vend);
    if (check)
      phase2_chunk_a<T, kMode, true>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2, nca2,
                                     tid, q);
    else
      phase2_chunk_a<T, kMode, false>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2,
                                      nca2, tid, q);
    if constexpr (kMode == 2) {
#pragma unroll
      for (int g = 0; g < kVA; ++g) q[g] = qn[g];
    }
    it.next();
    vbase = vend;
  }
}

// waits of the producer / epilogue warps back off with nanosleep so their
// polling does not steal issue slots from the consumer warps on the same SMSP
// Back-off (ns) of the producer's slot waits, the epilogue's partial waits and
// the consumers' broadcast waits; a negative value selects a try_wait with a
// suspend-time hint (the warp sleeps until the phase completes).
// Round 2 (profiles/r02_wait_park.txt): parking the producer's and the
// broadcast waits in the mbarrier (suspend-time hint) rather than re-polling
// every 64 ns, and letting the epilogue's cluster-scope partial wait spin,
// gives the headline +0.4 % on the same box (fewer issued instructions under
// the power cap).  CL = 1 keeps its spinning epilogue / broadcast waits.
#ifndef TG_SLEEP_PROD
#define TG_SLEEP_PROD -1
#endif
#ifndef TG_SLEEP_EPI
#define TG_SLEEP_EPI -1
#endif
#ifndef TG_SLEEP_BCAST
#define TG_SLEEP_BCAST -1
#endif
template <int kSleep>
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  if constexpr (kSleep < 0) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
  } else if constexpr (kSleep == 0) {
    while (!mbar_try_wait(bar, parity)) {
    }
  } else {
    while (!mbar_try_wait(bar, parity)) __nanosleep(kSleep);
  }
}

// Consumer warps of the fused anchor path: the same row loop as the default
// consumers (first row's prefix, phase 1, partial post to every CTA of the
// cluster, next row's prefix, phase 2), over z + za half-chunk pairs.
template <typename T, int CL, int kMode>
__device__ __forceinline__ void consumer_rows_a(const KParams& P, FusedSmemTail* tail,
                                                const RingBase& rb, const Slice& sl, int pre,
                                                int64_t cid, int64_t ncl, uint32_t rank,
                                                int warp, int lane, int tid) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  const int64_t NR = P.n_rows;
  const int V = int(P.vocab);
#ifdef TG_FUSED_PROF
  const long long t_start = clock64();
#endif
  typename AGeo<kMode>::It pos0 = {0u};
  AccA acc = acc_init_a();
  const uint64_t pol_q = policy_evict_first();  // mode 2: the anchor row's last use
  int vtid = tid;
  // (mode 3 with the copier: identity -- a TMEM column block's 128 lanes are
  // the 128 consecutive threads whose vectors one tcgen05.cp.128x128b moves)
  if constexpr (kConsumerWarps == 16 && !(kMode == 3 && kSplitCp)) {  // sub-partitions 2 / 3 first
    const int q = warp & 3, grp = warp >> 2;
    const int vw = (q >= 2) ? (grp * 2 + (q - 2)) : (8 + grp * 2 + q);
    vtid = vw * 32 + lane;
  }
  if (cid < NR) phase1_range_a<T, kMode>(acc, pos0, rb, sl, 0, pre, vtid);
  int64_t k = 0;
  for (int64_t row = cid; row < NR; row += ncl, ++k) {
    const int64_t nrow = row + ncl;
    const int y = __ldg(&P.target[row]);
    const int vy = (y >= 0 && y < V) ? (y / EPV) : -1;
    const int ye = (vy >= 0) ? y - vy * EPV : 0;
    const int par = int(k & 1);
    phase1_range_a<T, kMode>(acc, pos0, rb, sl, pre, sl.nchunk, vtid);
    float lq;
    const float4 o = warp_partial_a(acc, lq);
    if (lane == 0) {
      const int slot = int(rank) * kConsumerWarps + warp;
      tail->wpart[par][slot] = o;
      tail->wpart_q[par][slot] = lq;
      if constexpr (CL > 1) {
        const uint32_t la = smem_u32(&tail->wpart[par][slot]);
        const uint32_t lqa = smem_u32(&tail->wpart_q[par][slot]);
        const uint32_t lb = smem_u32(&tail->pbar[par]);
#pragma unroll
        for (int r = 0; r < CL; ++r)
          if (r != int(rank)) {
            st_async_v4(map_to_rank(la, r), o.x, o.y, o.z, o.w, map_to_rank(lb, r));
            st_async_f32(map_to_rank(lqa, r), lq, map_to_rank(lb, r));
          }
      }
      arrive_u32(smem_u32(&tail->pbar[par]));
    }
    typename AGeo<kMode>::It npos = pos0;
    npos.advance(sl.nchunk);
    acc_new_row_a(acc);
    if (nrow < NR) phase1_range_a<T, kMode>(acc, npos, rb, sl, 0, pre, vtid);
    {
      TG_PROF_T0();
      mbar_wait_u32<(CL == 1 ? 0 : TG_SLEEP_BCAST)>(smem_u32(&tail->bbar[par]),
                                                    uint32_t((k >> 1) & 1));
      TG_PROF_ADD(tail, 1);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const float4 bc = tail->bcast[par];
    const float ca = tail->bcast_ca[par];
    const float lseL = bc.z * kLog2e;
    const uint64_t nl2 = pk2(-lseL, -lseL), av2 = pk2(bc.x, bc.x), hz2 = pk2(bc.y, bc.y);
    const uint64_t nca2 = pk2(-ca, -ca);
    char* dzrow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
    const char* qrow = reinterpret_cast<const char*>(P.anchor) + row * P.ld_anchor * ESZ;
    phase2_row_a<T, kMode>(sl, pos0, rb, qrow, dzrow, vy, ye, bc.w, nl2, av2, hz2, nca2, vtid,
                           pol_q);
    pos0 = npos;
#ifdef TG_FUSED_PROF
    if (tid == 0) tail->prof[6] += 1;
#endif
  }
#ifdef TG_FUSED_PROF
  if (tid == 0) tail->prof[2] = (unsigned long long)(clock64() - t_start);
#endif
}

template <typename T, int CL, int kA = 0>
__global__ void __launch_bounds__(kFusedThreads, 1)
    k_fused_tma(const KParams P, const RowMeta* __restrict__ meta, int prefetch) {
  // prefetch: bits 0..15 L2 look-ahead in rows (bulk prefetch of whole row
  // slices), bits 16..31 (anchor mode 3) L2 look-ahead in stash positions
  const int prefetch_rows = prefetch & 0xFFFF;
  const uint32_t pf_chunks = uint32_t(prefetch) >> 16;
  // kA: 0 no anchor; 1 anchor KL with z and za in the TMEM stash; 2 anchor KL
  // with z in the stash and za re-read from L2 in phase 2 (twice the stash
  // columns per slot: Qwen-vocabulary rows fit 2-CTA clusters, all 148 SMs)
  static_assert(!kA || kStash, "the fused anchor path keeps the row slices in the TMEM stash");
  // kA: a ring / stash slot holds a z + za half-chunk pair
  constexpr int EPV = Vec<T>::N;  // elements per 16-byte vector
  constexpr int ESZ = elem_bytes<T>();
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem;
  FusedSmemTail* tail = reinterpret_cast<FusedSmemTail*>(smem + size_t(kSlots) * kChunk);
  const RingBase rb0 = {smem_u32(ring), smem_u32(&tail->full[0]), smem_u32(&tail->empty[0]), 0u,
                       smem_u32(&tail->tfull[0])};

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = (CL > 1) ? cluster_ctarank() : 0u;
  const int64_t cid = (CL > 1) ? int64_t(cluster_id_x()) : int64_t(blockIdx.x);
  const int64_t ncl = (CL > 1) ? int64_t(n_clusters_x()) : int64_t(gridDim.x);
  const int64_t NR = P.n_rows;
  const int V = int(P.vocab);

  // column slice of this CTA, in 16-byte vectors (32-bit: V < 2^31)
  Slice sl;
  const int nvec = (V + EPV - 1) / EPV;
  sl.v0 = int((int64_t(rank) * nvec) / CL);
  sl.v1 = int((int64_t(rank + 1) * nvec) / CL);
  const uint32_t slice_bytes = uint32_t(sl.v1 - sl.v0) * 16u;
  constexpr uint32_t kStep = kA ? AGeo<kA ? kA : 1>::HALF : uint32_t(kChunk);  // row bytes per slot
  constexpr int kRing = kA ? AGeo<kA ? kA : 1>::SLOTS : kSlots;
  using PIt = typename std::conditional<(kA == 3), typename AGeo<3>::It,
                                        RingItT<kRing, kA ? AGeo<kA ? kA : 1>::CHUNK
                                                          : uint32_t(kChunk)>>::type;
  sl.nchunk = int((slice_bytes + kStep - 1) / kStep);
  sl.tail_vec = (V % EPV) ? nvec - 1 : -1;  // global vector holding columns >= V
  sl.tail_valid = V - (nvec - 1) * EPV;
  // next-row phase-1 chunks that fit in the ring beside this row's slice
  const int pre = min(min(kMaxPrefixChunks,
                          (kStash ? (kA ? AGeo<kA ? kA : 1>::TSLOTS : kTSlots) : kSlots) -
                              sl.nchunk),
                      sl.nchunk);

  if (tid == 0) {
    // mode 3 with the copier: a landing slot is freed by the copy's commit
    constexpr bool kCp = kA == 3 && kSplitCp;
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], (kCp && i < kLSlots) ? 1
                                 : (kA == 3 && kArriveAll) ? kConsumers : kConsumerWarps);
    }
    if constexpr (kCp) {
      for (int i = 0; i < kTSlots; ++i) {
        mbar_init(&tail->tfull[i], 1);
        mbar_init(&tail->tempty[i], kConsumerWarps);
      }
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tail->pbar[i], kConsumerWarps + (CL > 1 ? 1 : 0));  // + epilogue expect_tx
      mbar_init(&tail->bbar[i], kArriveAll ? 32 : 1);
    }
    fence_mbar_init();
#ifdef TG_FUSED_PROF
    for (int i = 0; i < 16; ++i) tail->prof[i] = 0ull;
    for (int i = 0; i < 2; ++i) {
      tail->post_first[i] = ~0ull;
      tail->post_last[i] = 0ull;
    }
#endif
  }
  if constexpr (kStash) {
    if (warp == kProducerWarp) {  // one full warp allocates (and later frees) the stash
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&tail->tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  // every CTA is resident: the tail kernel (PDL) may be scheduled; it waits
  // for this grid's completion itself
  if (tid == 0) pdl_trigger();
  if (CL > 1)
    cluster_sync_all();
  else
    __syncthreads();
  RingBase rb = rb0;
  if constexpr (kStash) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    rb.tmem = tail->tmem_base + ((uint32_t(32 * (warp & 3))) << 16) + uint32_t(warp >> 2) * 128u;
  }
#ifdef TG_FUSED_PROF
  const long long t_start = clock64();
#endif

  if (warp == kProducerWarp) {
    // ===================== producer warp: bulk TMA into the ring =====================
    // mode 3: lane 0 issues the TMEM positions (landing slots), lane 1 the
    // shared stash positions -- two in-order issuers, so a stash slot still
    // held by phase 2 does not hold up the landing slots' read-ahead
    if (lane < (kA == 3 ? 2 : 1) && sl.nchunk > 0) {
      const uint64_t pol = policy_evict_first();
      // mode 2: the anchor row stays in L2 until phase 2 re-reads it
      const uint64_t pol_q = policy_za();
      const char* base = reinterpret_cast<const char*>(P.logits);
      auto slice_ptr = [&](int64_t row) {
        const int64_t src_row = P.row_index ? P.row_index[row] : row;
        return base + src_row * P.ld * ESZ + int64_t(sl.v0) * 16;
      };
      for (int i = 0; i < prefetch_rows && lane == 0; ++i) {
        const int64_t r = cid + int64_t(i) * ncl;
        if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
      }
      PIt it = {0u};
      uint32_t pc = 0;  // mode 3: next position to prefetch into L2
      for (int64_t row = cid; row < NR; row += ncl) {
        if (prefetch_rows > 0 && lane == 0) {
          const int64_t r = row + int64_t(prefetch_rows) * ncl;
          if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
        }
        const char* src = slice_ptr(row);
        for (int j = 0; j < sl.nchunk; ++j) {
          // L2 look-ahead by positions (anchor mode 3: the landing slots hold
          // only a few pairs, so the pairs behind them are pulled into L2
          // early and their TMA loads then see L2 latency)
          if (lane == 0 && pf_chunks > 0) {
            for (; pc < it.c + pf_chunks; ++pc) {
              const int64_t prow = cid + int64_t(pc / uint32_t(sl.nchunk)) * ncl;
              if (prow >= NR) break;
              const uint32_t poff = (pc % uint32_t(sl.nchunk)) * kStep;
              const uint32_t pb = min(kStep, slice_bytes - poff);
              prefetch_l2(slice_ptr(prow) + poff, pb);
              if constexpr (kA != 0)
                prefetch_l2(reinterpret_cast<const char*>(P.anchor) + prow * P.ld_anchor * ESZ +
                                int64_t(sl.v0) * 16 + poff,
                            pb);
            }
          }
          if constexpr (kA == 3) {
            if (it.in_tmem() != (lane == 0)) {  // the other issuer's position
              it.next();
              continue;
            }
          }
          {
            TG_PROF_T0();
            // (CL = 1, short rows: the 64 ns re-poll measured 0.9 % faster)
            mbar_wait_u32<(CL == 1 ? 64 : TG_SLEEP_PROD)>(it.empty(rb), it.phase() ^ 1u);
            TG_PROF_ADD(tail, 3);
          }
          // kA: a half chunk of z and the same columns of the anchor row in one slot
          const uint32_t step = kStep;
          const uint32_t off = uint32_t(j) * step;
          const uint32_t bytes = min(step, slice_bytes - off);
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                           it.full(rb)),
                       "r"(kA ? 2 * bytes : bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1], %2, [%3], %4;" ::"r"(it.addr(rb)),
              "l"(src + off), "r"(bytes), "r"(it.full(rb)), "l"(pol)
              : "memory");
          if constexpr (kA) {
            const char* qsrc = reinterpret_cast<const char*>(P.anchor) +
                               row * P.ld_anchor * ESZ + int64_t(sl.v0) * 16;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1], %2, [%3], %4;" ::"r"(it.addr(rb) + kStep),
                "l"(qsrc + off), "r"(bytes), "r"(it.full(rb)), "l"(kA == 2 ? pol_q : pol)
                : "memory");
          }
          it.next();
        }
      }
    }
    if constexpr (kA == 3 && kSplitCp) {
      // ---- copier lane (mode 3): landed TMEM-position pairs -> TMEM (tcgen05.cp) ----
      if (lane == 2 && sl.nchunk > 0) {
        PIt it = {0u};
        const uint32_t tb = tail->tmem_base;  // lane 0, column 0 of the CTA's 512 columns
        for (int64_t row = cid; row < NR; row += ncl) {
          for (int j = 0; j < sl.nchunk; ++j) {
            if (it.in_tmem()) {
#ifdef TG_FUSED_PROF
              const long long c0 = clock64();
#endif
              mbar_wait_u32<TG_SLEEP_PROD>(it.tempty(rb), it.tphase() ^ 1u);
#ifdef TG_FUSED_PROF
              const long long c1 = clock64();
#endif
              mbar_wait_u32<0>(it.full(rb), it.phase());
#ifdef TG_FUSED_PROF
              tail->prof[13] += (unsigned long long)(c1 - c0);
              tail->prof[14] += (unsigned long long)(clock64() - c1);
#endif
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint32_t src = it.addr(rb);
              const uint32_t dst = tb + it.pos() * uint32_t(kTCols);
              // column block cb = warps 4 cb .. 4 cb + 3 = threads 128 cb .. + 127;
              // vector v of every thread: z g = 0 / 1, za g = 0 / 1
#pragma unroll
              for (int cb = 0; cb < 4; ++cb)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                  tmem_cp_128x128b(dst + uint32_t(cb) * 128u + uint32_t(v) * 4u,
                                   src + (v >= 2 ? kStep : 0u) + uint32_t(v & 1) * kConsumers * 16u +
                                       uint32_t(cb) * 128u * 16u);
              tc_commit(it.tfull(rb));  // the consumers may read the position
              tc_commit(it.empty(rb));  // the landing slot may be refilled
            }
            it.next();
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kEpilogueWarp) {
    // ===================== epilogue warp: row reductions + registry epilogue ==========
    // Off the consumers' critical path: while it reduces row k, exchanges with
    // the cluster peers and evaluates the loss terms, the consumers already run
    // phase 1 of row k+1.
    // The group prologue (k_counts_prep) may still run (PDL): the producer and
    // the consumers already stream the first rows; the row metadata it writes
    // (advantages, weights) is read here only after it completed.
    pdl_wait();
    double sd[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) sd[i] = 0.0;
    double sd_a[2] = {0.0, 0.0};  // kA: anchor loss, Sigma KL(p || q)
    // the row's metadata and target logit are fetched one row ahead (after the
    // previous row's broadcast), so their dependent loads stay off the path
    //
    // The target logit is read from global memory only by the CTA whose slice
    // holds it (and sent to the peers with the partials): with dlogits written
    // in place, a peer's phase 2 may overwrite that column as soon as its own
    // broadcast of the row went out, while the owner's phase 2 comes after its
    // own broadcast, which needs this load.
    int seq_cur = (lane == 0 && cid < NR) ? seq_of_row(P, cid) : 0;
    RowMeta nxt;
    float nzy = kNegInf;
    // CTA rank whose column slice holds the target vector (-1: no valid target)
    auto owner_of = [&](int y) {
      if (y < 0 || y >= V) return -1;
      const int vyv = y / EPV;
      int own = 0;
#pragma unroll
      for (int q = 1; q < CL; ++q)
        if (int((int64_t(q) * nvec) / CL) <= vyv) own = q;
      return own;
    };
    auto fetch = [&](int64_t r, int parr) {
      nxt = row_meta(P, r, seq_cur);
      nzy = kNegInf;  // raw, unclamped target logit
      if (owner_of(nxt.y) == int(rank)) {
        const int64_t src_row = P.row_index ? P.row_index[r] : r;
        nzy = Vec<T>::load1(reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ, nxt.y);
        if constexpr (CL > 1) {
          const uint32_t za = smem_u32(&tail->zy[parr]), zb = smem_u32(&tail->pbar[parr]);
#pragma unroll
          for (int q = 0; q < CL; ++q)
            if (q != int(rank)) st_async_f32(map_to_rank(za, q), nzy, map_to_rank(zb, q));
        }
      }
    };
    if (lane == 0 && cid < NR) fetch(cid, 0);
    int64_t k = 0;
    for (int64_t row = cid; row < NR; row += ncl, ++k) {
      const int par = int(k & 1);
      const uint32_t parity = uint32_t((k >> 1) & 1);
      const RowMeta cur = nxt;
      float tzy = nzy;
      int own = 0;
      if (lane == 0) {
        own = owner_of(cur.y);
        if constexpr (CL > 1)
          mbar_arrive_expect_tx(&tail->pbar[par], (CL - 1) * kConsumerWarps * (kA ? 20 : 16) +
                                                      (own >= 0 && own != int(rank) ? 4 : 0));
      }
      {
        TG_PROF_T0();
        if constexpr (CL > 1)
          mbar_wait_cluster_sleep<TG_SLEEP_EPI>(smem_u32(&tail->pbar[par]), parity);
        else  // short rows (CL = 1): spin, the waits are frequent and short (+0.65 %)
          mbar_wait_u32<0>(smem_u32(&tail->pbar[par]), parity);
        TG_PROF_ADD(tail, 4);
      }
#ifdef TG_FUSED_PROF
      const long long t_crit = clock64();
      const long long t_xdone = t_crit;
      if (lane == 0) {
        tail->prof[9] += (unsigned long long)t_crit - tail->post_first[par];
        tail->prof[10] += tail->post_last[par] - tail->post_first[par];
        tail->post_first[par] = ~0ull;
        tail->post_last[par] = 0ull;
      }
#endif
      // all CL x warps partials, merged in a fixed lane order: lane 0 holds the
      // same bits on every CTA of the cluster
      constexpr int NP = CL * kConsumerWarps;
      // (m, Sigma e, Sigma e z[, Sigma e (z - za)]) of the row; kA: the anchor's
      // log-sum-exp from the per-warp ones
      constexpr bool kRedux = TG_MERGE_REDUX && kA && NP > 32;
      const float4 tot4 = kRedux ? merge_partials<NP, (kA != 0)>(tail->wpart[par], lane)
                                 : merge_partials_online<NP, (kA != 0)>(tail->wpart[par], lane);
      const Online tot = {tot4.x, tot4.y, tot4.z};
      float lseq = 0.f;
      if constexpr (kA)
        lseq = kRedux ? merge_lse<NP>(tail->wpart_q[par], lane)
                      : merge_lse_online<NP>(tail->wpart_q[par], lane);
      // sanitizer build: every lane that read the partials releases them
      if (kArriveAll && lane != 0) arrive_u32(smem_u32(&tail->bbar[par]));
      if (lane == 0) {
        // fast log / divide on the critical path; full precision when the row's
        // lp feeds sequence sums that couple the gradient (route 4) or the
        // anchor KL takes a difference of log-sum-exps, as in k_fwd / k_fwd_tma
        const bool precise = kA != 0 || (P.flags & TG_FLAG_UNSCALED_GRAD) != 0;
        const float lse = tot.m + (precise ? logf(tot.s) : __logf(tot.s));
        const float H = lse - (precise ? tot.t / tot.s : __fdividef(tot.t, tot.s));
        const bool bad_target = (cur.flags & 2u) != 0;
        if (CL > 1 && own >= 0 && own != int(rank)) tzy = tail->zy[par];
        const float lp = tzy - lse;
        RowTerms o;
        if (P.flags & TG_FLAG_UNSCALED_GRAD) {  // coupled, one pass: dz = p - e, scale later
          o = RowTerms{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0, 0, 0};
        } else {
          o = meta_terms(P, cur, lp, H);
        }
        if (bad_target) {
          o.s = 0.f;
          o.h = 0.f;
        }
        float ca = 0.f, akl = 0.f, a_anchor = 0.f;
        if constexpr (kA) {  // k_rowcoef's anchor terms: KL(p || q) = Sigma p (z - za) - lse + lse_q
          akl = tot4.w / tot.s - lse + lseq;
          ca = bad_target ? 0.f : cur.ca;
          a_anchor = ca * (lse - lseq + akl);
          tail->bcast_ca[par] = ca;
        }
        tail->bcast[par] = make_float4(o.s + o.h * (H - lse) - a_anchor, o.h + ca, lse, o.s);
        arrive_u32(smem_u32(&tail->bbar[par]));
        if (row + ncl < NR) fetch(row + ncl, par ^ 1);
#ifdef TG_FUSED_PROF
        tail->prof[7] += (unsigned long long)(clock64() - t_crit);
        tail->prof[8] += (unsigned long long)(clock64() - t_xdone);
#endif
        if (rank == 0) {  // outputs + statistics, after the broadcast
          P.lp[row] = lp;
          P.ent[row] = H;
          P.lse[row] = lse;
          const bool nonfin = !(finite_f(lse) && finite_f(lp) && finite_f(H) && finite_f(o.s) &&
                                finite_f(o.h) && finite_f(a_anchor));
          if constexpr (kA) {
            sd_a[0] += double(ca) * double(akl);
            sd_a[1] += akl;
          }
          sd[0] += o.l_pg;
          sd[1] += o.l_kl;
          sd[2] += o.l_ent;
          sd[3] += o.l_sft;
          sd[4] += o.clipped;
          sd[5] += o.dual;
          if (o.rl) {
            sd[6] += H;
            sd[7] += o.kl;
            sd[8] += o.ppo_kl;
            sd[11] += o.ratio;
            sd[12] += 1.0;
          }
          sd[9] += lp;
          sd[10] += nonfin;
          sd[13] += bad_target;
          sd[14] += 1.0;
        }
      }
    }
    // rank 0 of each cluster accumulated its rows; other ranks store zeros
    if (lane == 0) {
      double* dst = P.partials + size_t(blockIdx.x) * TG_NSTAT;
      for (int i = 0; i < TG_NSTAT; ++i) dst[i] = 0.0;
      dst[TG_S_PG_LOSS] = sd[0];
      dst[TG_S_KL_LOSS] = sd[1];
      dst[TG_S_ENTROPY_LOSS] = sd[2];
      dst[TG_S_SFT_LOSS] = sd[3];
      dst[TG_S_CLIP_COUNT] = sd[4];
      dst[TG_S_DUAL_CLIP_COUNT] = sd[5];
      dst[TG_S_SUM_ENTROPY] = sd[6];
      dst[TG_S_SUM_KL] = sd[7];
      dst[TG_S_SUM_PPO_KL] = sd[8];
      dst[TG_S_SUM_LP] = sd[9];
      dst[TG_S_NONFINITE] = sd[10];
      dst[TG_S_SUM_RATIO] = sd[11];
      dst[TG_S_N_TOK_RL] = sd[12];
      dst[TG_S_INVALID] = sd[13];
      dst[TG_S_N_TOK] = sd[14];
      dst[TG_S_ANCHOR_LOSS] = sd_a[0];
      dst[TG_S_SUM_ANCHOR_KL] = sd_a[1];
    }
  } else if (kA != 0 && warp < kConsumerWarps) {
    consumer_rows_a<T, CL, kA>(P, tail, rb, sl, pre, cid, ncl, rank, warp, lane, tid);
  } else if (warp < kConsumerWarps) {
    // ===================== consumer warps =====================
    RingIt pos0 = {0u};  // the current row's first chunk
    Acc1 acc = acc_init();
#ifndef TG_WM_ALL
#define TG_WM_ALL 1
#endif
    constexpr bool kWM = CL == 1 || TG_WM_ALL;  // warp-uniform reference max
    // Virtual thread index for the chunk layout: the warps of SM sub-partitions
    // 2 and 3 come first, so a partial last chunk's valid vectors go to them --
    // sub-partitions 0 and 1 also host the epilogue and producer warps.  (Any
    // permutation is valid: each thread stashes its own data in its own TMEM
    // lane and phase 2 uses the same mapping.)
#ifndef TG_VWARP_PERM
#define TG_VWARP_PERM 1
#endif
    int vtid = tid;
    if constexpr (TG_VWARP_PERM && kConsumerWarps == 16) {
      const int q = warp & 3, grp = warp >> 2;
      const int vw = (q >= 2) ? (grp * 2 + (q - 2)) : (8 + grp * 2 + q);
      vtid = vw * 32 + lane;
    }
    if (cid < NR) phase1_range<T, kWM>(acc, pos0, rb, sl, 0, pre, vtid);  // first row's prefix
    int y_cur = (cid < NR) ? __ldg(&P.target[cid]) : 0;
    int64_t k = 0;
    for (int64_t row = cid; row < NR; row += ncl, ++k) {
      const int64_t nrow = row + ncl;
      const int y_next = (nrow < NR) ? __ldg(&P.target[nrow]) : 0;  // prefetch
      const int y = y_cur;
      const int vy = (y >= 0 && y < V) ? (y / EPV) : -1;  // global vector holding the target
      const int ye = (vy >= 0) ? y - vy * EPV : 0;
      const int par = int(k & 1);

      // ---------------- phase 1 (rest of the row) ----------------
      phase1_range<T, kWM>(acc, pos0, rb, sl, pre, sl.nchunk, vtid);
      const Online o = warp_partial<kWM>(acc);
      if (lane == 0) {
        // the warp partial goes to every CTA of the cluster (peers: DSMEM st.async
        // completing tx bytes on their partials barrier), so each epilogue merges
        // all CL x warps partials after a single wait
        const int slot = int(rank) * kConsumerWarps + warp;
#ifdef TG_FUSED_PROF
        const unsigned long long tpost = clock64();
        atomicMin(&tail->post_first[par], tpost);
        atomicMax(&tail->post_last[par], tpost);
#endif
        tail->wpart[par][slot] = make_float4(o.m, o.s, o.t, 0.f);
        if constexpr (CL > 1) {
          const uint32_t la = smem_u32(&tail->wpart[par][slot]);
          const uint32_t lb = smem_u32(&tail->pbar[par]);
#pragma unroll
          for (int r = 0; r < CL; ++r)
            if (r != int(rank)) st_async_v4(map_to_rank(la, r), o.m, o.s, o.t, 0.f, map_to_rank(lb, r));
        }
        arrive_u32(smem_u32(&tail->pbar[par]));
      }
      // ---------------- phase 1 prefix of the next row (hides the epilogue) ----------
      RingIt npos = pos0;
      npos.advance(sl.nchunk);
      acc_new_row(acc);
      if (nrow < NR) phase1_range<T, kWM>(acc, npos, rb, sl, 0, pre, vtid);

      // ---------------- phase 2: dz from the resident slice ----------------
      {
        TG_PROF_T0();
        mbar_wait_u32<(CL == 1 ? 0 : TG_SLEEP_BCAST)>(smem_u32(&tail->bbar[par]),
                                                      uint32_t((k >> 1) & 1));
        TG_PROF_ADD(tail, 1);
      }
      if constexpr (kStash) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      const float4 bc = tail->bcast[par];
      const float a = bc.x, hz = bc.y, s_t = bc.w;
      const float lseL = bc.z * kLog2e;
      const uint64_t nl2 = pk2(-lseL, -lseL), av2 = pk2(a, a), hz2 = pk2(hz, hz);
      char* dzrow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
      if (hz == 0.f)
        phase2_row<T, false>(sl, pos0, rb, dzrow, vy, ye, s_t, nl2, av2, hz2, vtid, lane);
      else
        phase2_row<T, true>(sl, pos0, rb, dzrow, vy, ye, s_t, nl2, av2, hz2, vtid, lane);
      pos0 = npos;
      y_cur = y_next;
#ifdef TG_FUSED_PROF
      if (tid == 0) tail->prof[6] += 1;
#endif
    }
#ifdef TG_FUSED_PROF
    if (tid == 0) tail->prof[2] = (unsigned long long)(clock64() - t_start);
#endif
  }
  if (CL > 1)
    cluster_sync_all();  // no CTA leaves while a peer may still st.async into it
  if constexpr (kStash) {
    if (CL == 1) __syncthreads();
    if (warp == kProducerWarp) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tail->tmem_base)
                   : "memory");
    }
  }
#ifdef TG_FUSED_PROF
  __syncthreads();
  if (tid < 16) g_fused_prof[blockIdx.x][tid] = tail->prof[tid];
#endif
}

// ---------------------------------------------------------------------------
// k_fwd_tma: forward-only streaming logprob (tg_logprob_fwd, and the forward
// pass of the two-pass / sequence-coupled routes).  Same warp roles and ring
// as k_fused_tma, but nothing has to stay resident: each chunk is released as
// soon as its phase-1 sums are taken, so the whole 224 KB ring is read-ahead,
// one CTA owns whole rows (no cluster), and the consumers never wait for the
// epilogue -- it only merges the warp partials, reads the target logit and
// writes lse / lp / entropy.  2V bytes read per row.

constexpr int kFwdPar = 4;  // row-partial buffers between the consumers and the epilogue

struct FwdSmemTail {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t pbar[kFwdPar];  // consumers -> epilogue: partials of a row written
  uint64_t ebar[kFwdPar];  // epilogue -> consumers: partial buffer free again
  float4 wpart[kFwdPar][kConsumerWarps];
};

template <typename T>
__device__ __forceinline__ void phase1_stream_row(Acc1& acc, RingIt& it, const RingBase& rb,
                                                  const Slice& sl, int tid, int lane) {
  int vbase = sl.v0;
  for (int c = 0; c < sl.nchunk; ++c) {
    const uint32_t empty = it.empty(rb);
    const int vend = vbase + kVecPerChunk;
    const bool has_tail = sl.tail_vec >= vbase && sl.tail_vec < vend;
    if (vend <= sl.v1 && !has_tail)
      phase1_chunk<T, false, false>(acc, it, rb, vbase, sl, tid);
    else if (!has_tail)
      phase1_chunk<T, true, false>(acc, it, rb, vbase, sl, tid);
    else
      phase1_chunk<T, true, true>(acc, it, rb, vbase, sl, tid);
    __syncwarp();
    if (lane == 0) arrive_u32(empty);  // the chunk's data is in registers: slot free
    vbase = vend;
  }
}

template <typename T>
__global__ void __launch_bounds__(kFusedThreads, 1) k_fwd_tma(const KParams P) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  extern __shared__ __align__(1024) unsigned char smem[];
  FwdSmemTail* tail = reinterpret_cast<FwdSmemTail*>(smem + size_t(kSlots) * kChunk);
  const RingBase rb = {smem_u32(smem), smem_u32(&tail->full[0]), smem_u32(&tail->empty[0])};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t NR = P.n_rows;
  const int V = int(P.vocab);
  Slice sl;
  const int nvec = (V + EPV - 1) / EPV;
  sl.v0 = 0;
  sl.v1 = nvec;
  const uint32_t row_bytes = uint32_t(nvec) * 16u;
  sl.nchunk = int((row_bytes + kChunk - 1) / kChunk);
  sl.tail_vec = (V % EPV) ? nvec - 1 : -1;
  sl.tail_valid = V - (nvec - 1) * EPV;

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], kConsumerWarps);
    }
    for (int i = 0; i < kFwdPar; ++i) {
      mbar_init(&tail->pbar[i], kConsumerWarps);
      mbar_init(&tail->ebar[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    if (lane == 0 && sl.nchunk > 0) {
      const uint64_t pol = policy_evict_first();
      const char* base = reinterpret_cast<const char*>(P.logits);
      RingIt it = {0u};
      for (int64_t row = blockIdx.x; row < NR; row += gridDim.x) {
        const int64_t src_row = P.row_index ? P.row_index[row] : row;
        const char* src = base + src_row * P.ld * ESZ;
        for (int j = 0; j < sl.nchunk; ++j) {
          mbar_wait_u32<TG_SLEEP_PROD>(it.empty(rb), it.phase() ^ 1u);
          const uint32_t off = uint32_t(j) * kChunk;
          const uint32_t bytes = min(uint32_t(kChunk), row_bytes - off);
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                           it.full(rb)),
                       "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1], %2, [%3], %4;" ::"r"(it.addr(rb)),
              "l"(src + off), "r"(bytes), "r"(it.full(rb)), "l"(pol)
              : "memory");
          it.next();
        }
      }
    }
    __syncwarp();
  } else if (warp == kEpilogueWarp) {
    int64_t k = 0;
    for (int64_t row = blockIdx.x; row < NR; row += gridDim.x, ++k) {
      const int slot = int(k % kFwdPar);
      const uint32_t parity = uint32_t((k / kFwdPar) & 1);
      float zy = kNegInf;  // target logit, read ahead of the wait
      if (lane == 0) {
        const int y = P.target[row];
        if (y >= 0 && y < V) {
          const int64_t src_row = P.row_index ? P.row_index[row] : row;
          zy = Vec<T>::load1(reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ, y);
        }
      }
      mbar_wait_u32<TG_SLEEP_EPI>(smem_u32(&tail->pbar[slot]), parity);
      Online acc_p = {kNegInf, 0.f, 0.f};
      if (lane < kConsumerWarps) {
        const float4 v = tail->wpart[slot][lane];
        acc_p = Online{v.x, v.y, v.z};
      }
      __syncwarp();
      if (lane == 0) arrive_u32(smem_u32(&tail->ebar[slot]));
      const Online tot = warp_merge_first<kConsumerWarps>(acc_p);
      if (lane == 0) {  // off the consumers' path: full-precision log and divide
        const float lse = tot.m + logf(tot.s);
        P.lse[row] = lse;
        P.lp[row] = zy - lse;
        P.ent[row] = lse - tot.t / tot.s;
      }
    }
  } else if (warp < kConsumerWarps) {
    RingIt it = {0u};
    Acc1 acc = acc_init();
    int64_t k = 0;
    for (int64_t row = blockIdx.x; row < NR; row += gridDim.x, ++k) {
      acc_new_row(acc);
      phase1_stream_row<T>(acc, it, rb, sl, tid, lane);
      const Online o = warp_partial<false>(acc);
      const int slot = int(k % kFwdPar);
      if (lane == 0) {
        if (k >= kFwdPar)  // the epilogue has read this buffer's previous row
          mbar_wait_u32<TG_SLEEP_BCAST>(smem_u32(&tail->ebar[slot]),
                                        uint32_t(((k / kFwdPar) - 1) & 1));
        tail->wpart[slot][warp] = make_float4(o.m, o.s, o.t, 0.f);
        arrive_u32(smem_u32(&tail->pbar[slot]));
      }
    }
  }
}

size_t fwd_tma_smem_bytes() { return size_t(kSlots) * kChunk + sizeof(FwdSmemTail); }

cudaError_t launch_fwd_tma(const KParams& P, int n_sms, cudaStream_t stream) {
#ifdef TG_FUSED_PROF
  return cudaErrorNotSupported;  // the profiling counters assume k_fused_tma's layout
#endif
  const size_t smem = fwd_tma_smem_bytes();
  const int64_t grid64 = P.n_rows < n_sms ? P.n_rows : n_sms;
  if (grid64 <= 0) return cudaSuccess;
  cudaError_t e;
  if (P.dtype == TG_DTYPE_BF16) {
    e = cudaFuncSetAttribute(k_fwd_tma<bf16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
    if (e != cudaSuccess) return e;
    k_fwd_tma<bf16_t><<<int(grid64), kFusedThreads, smem, stream>>>(P);
  } else {
    e = cudaFuncSetAttribute(k_fwd_tma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
    if (e != cudaSuccess) return e;
    k_fwd_tma<float><<<int(grid64), kFusedThreads, smem, stream>>>(P);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host-side launch helper (called from tg_api.cu)

size_t fused_smem_bytes(int n_slots) { return size_t(n_slots) * kChunk + sizeof(FusedSmemTail); }

template <typename T, int CL, int kA = 0>
static cudaError_t launch_fused_t(const KParams& P, const RowMeta* meta, int n_ctas,
                                  int prefetch_rows, cudaStream_t stream) {
  const size_t smem = fused_smem_bytes(kSlots);
  cudaError_t e = cudaFuncSetAttribute(k_fused_tma<T, CL, kA>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // PDL: start streaming rows while k_counts_prep (already resident: it
  // triggers on entry) finishes; only the epilogue warp waits for it
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_fused_tma<T, CL, kA>, P, meta, prefetch_rows);
}

cudaError_t launch_fused(const KParams& P, const void* meta, int cl, int amode, int n_slots,
                         int n_ctas, int prefetch_rows, cudaStream_t stream) {
  if (n_slots != kSlots) return cudaErrorInvalidValue;
  const RowMeta* m = reinterpret_cast<const RowMeta*>(meta);
  if (P.anchor && P.anchor_beta > 0.f) {  // fused anchor KL (fused_plan's anchor rules)
    if (amode == 3) {  // split stash: TMEM + shared-memory positions
      if (P.dtype == TG_DTYPE_BF16 && cl == 2)
        return launch_fused_t<bf16_t, 2, 3>(P, m, n_ctas, prefetch_rows, stream);
      if (P.dtype != TG_DTYPE_BF16 && cl == 4)
        return launch_fused_t<float, 4, 3>(P, m, n_ctas, prefetch_rows, stream);
      return cudaErrorInvalidValue;
    }
    if (amode == 2) {  // z stashed, za re-read from L2
      if (P.dtype == TG_DTYPE_BF16) {
        if (cl == 1) return launch_fused_t<bf16_t, 1, 2>(P, m, n_ctas, prefetch_rows, stream);
        if (cl == 2) return launch_fused_t<bf16_t, 2, 2>(P, m, n_ctas, prefetch_rows, stream);
      } else {
        if (cl == 2) return launch_fused_t<float, 2, 2>(P, m, n_ctas, prefetch_rows, stream);
        if (cl == 4) return launch_fused_t<float, 4, 2>(P, m, n_ctas, prefetch_rows, stream);
      }
      return cudaErrorInvalidValue;
    }
    if (P.dtype == TG_DTYPE_BF16) {
      if (cl == 1) return launch_fused_t<bf16_t, 1, 1>(P, m, n_ctas, prefetch_rows, stream);
      if (cl == 2) return launch_fused_t<bf16_t, 2, 1>(P, m, n_ctas, prefetch_rows, stream);
      if (cl == 3) return launch_fused_t<bf16_t, 3, 1>(P, m, n_ctas, prefetch_rows, stream);
      if (cl == 4) return launch_fused_t<bf16_t, 4, 1>(P, m, n_ctas, prefetch_rows, stream);
    } else {  // fp32 rows: the slices fit the stash up to V ~ 65 k (CL <= 4)
      if (cl == 1) return launch_fused_t<float, 1, 1>(P, m, n_ctas, prefetch_rows, stream);
      if (cl == 2) return launch_fused_t<float, 2, 1>(P, m, n_ctas, prefetch_rows, stream);
      if (cl == 4) return launch_fused_t<float, 4, 1>(P, m, n_ctas, prefetch_rows, stream);
    }
    return cudaErrorInvalidValue;
  }
  if (P.dtype == TG_DTYPE_BF16) {
    if (cl == 1) return launch_fused_t<bf16_t, 1>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 2) return launch_fused_t<bf16_t, 2>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 3) return launch_fused_t<bf16_t, 3>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 4) return launch_fused_t<bf16_t, 4>(P, m, n_ctas, prefetch_rows, stream);
  } else {
    if (cl == 1) return launch_fused_t<float, 1>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 2) return launch_fused_t<float, 2>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 3) return launch_fused_t<float, 3>(P, m, n_ctas, prefetch_rows, stream);
    if (cl == 4) return launch_fused_t<float, 4>(P, m, n_ctas, prefetch_rows, stream);
  }
  return cudaErrorInvalidValue;
}

// Clusters of `cl` fused CTAs that can be co-resident (the kernel is persistent:
// a grid larger than this would run a second wave).  0 on error.
template <typename T, int CL>
static int max_clusters_t() {
  const size_t smem = fused_smem_bytes(kSlots);
  if (cudaFuncSetAttribute(k_fused_tma<T, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem)) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_fused_tma<T, CL>, &cfg) != cudaSuccess) return 0;
  return n;
}

static int fused_max_clusters_uncached(int dtype, int cl) {
  if (dtype == TG_DTYPE_BF16) {
    if (cl == 1) return max_clusters_t<bf16_t, 1>();
    if (cl == 2) return max_clusters_t<bf16_t, 2>();
    if (cl == 3) return max_clusters_t<bf16_t, 3>();
    if (cl == 4) return max_clusters_t<bf16_t, 4>();
  } else {
    if (cl == 1) return max_clusters_t<float, 1>();
    if (cl == 2) return max_clusters_t<float, 2>();
    if (cl == 3) return max_clusters_t<float, 3>();
    if (cl == 4) return max_clusters_t<float, 4>();
  }
  return 0;
}

// cached per (device, dtype, cluster size): the occupancy query is slow
int fused_max_clusters(int dtype, int cl) {
  static std::mutex mu;
  static int cache[64][2][5];
  static bool have[64][2][5] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || cl < 1 || cl > 4) return fused_max_clusters_uncached(dtype, cl);
  const int di = dtype == TG_DTYPE_BF16 ? 0 : 1;
  std::lock_guard<std::mutex> lk(mu);
  if (!have[dev][di][cl]) {
    cache[dev][di][cl] = fused_max_clusters_uncached(dtype, cl);
    have[dev][di][cl] = true;
  }
  return cache[dev][di][cl];
}

#ifdef TG_FUSED_PROF
// profiling build: per-CTA counters of the last fused launch (see prof[] above)
extern "C" int tg_debug_fused_prof(unsigned long long* out, int n_ctas) {
  if (n_ctas > 1024) n_ctas = 1024;
  return int(cudaMemcpyFromSymbol(out, g_fused_prof, size_t(n_ctas) * 16 * sizeof(unsigned long long)));
}
#endif

int fused_chunk_bytes() { return kChunk; }
int fused_max_slots() { return kSlots; }
// chunks of a row slice (+ look-ahead) that can stay resident: the shared-memory
// ring, or with the TMEM stash the per-warp TMEM ring
int fused_resident_chunks() { return kStash ? kTSlots : kSlots; }
// anchor mode 2 (z-only stash slots)
int fused_resident_chunks_z() { return kStash ? kTSlotsZ : 0; }
// anchor mode 3 (TMEM + shared-memory stash positions)
int fused_resident_chunks_split() { return kStash ? kTSlots + kSSlots : 0; }
// bytes of the row per ring slot in each anchor mode (z half of a z + za slot)
int fused_anchor_half_bytes(int) { return int(AGeo<1>::HALF); }
size_t rowmeta_bytes() { return sizeof(RowMeta); }

}  // namespace tg
