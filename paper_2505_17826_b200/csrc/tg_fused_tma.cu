// tg_fused_tma.cu -- K1: fused single-pass logprob + loss + dlogits over [T, V] logits.
//
// Replaces, per trainable row, policy.logprob (policy.py:194-212),
// policy.grad_logprob (policy.py:253-270) and the per-variant axpy of the
// loss's coefficient (algorithms.py:240-242, 263-266) -- plus the north_star
// PPO clip / KL / entropy terms -- with one read of the row from HBM and one
// write of d loss / d logits (4V bytes per row, the HBM roofline minimum).
//
// Design (B200-first):
//  * A thread-block cluster of CL CTAs (CL = 1 for V <= ~110k bf16, 2 for
//    Qwen's 151,936) owns one row at a time; CTA rank r owns a contiguous
//    column slice of the row.  The slice never leaves the SM: a producer warp
//    streams it into an 8-slot shared-memory ring (28 KB chunks, 224 KB) with
//    1-D bulk TMA (cp.async.bulk ... mbarrier::complete_tx), a full / empty
//    mbarrier pair per slot, and prefetches upcoming rows' slices into L2
//    (cp.async.bulk.prefetch.L2).
//  * 14 consumer warps, four 16-byte vectors per thread per chunk.  Phase 1
//    (as chunks land): online max / sum-exp / sum p*z in packed fp32x2
//    arithmetic (FFMA2 / FADD2) with MUFU ex2; -inf logits are clamped to
//    -1e30 with packed bf16x2 max; the running max is updated lazily behind a
//    warp vote.  Each warp posts its partial and arrives on an mbarrier.
//  * A dedicated epilogue warp merges the partials, reads the target logit
//    from the resident chunk, exchanges the CTA partial with its cluster peers
//    through DSMEM (st.async completing tx bytes on the peer's mbarrier;
//    rank-order merge => bit-identical lse on every CTA), evaluates the
//    registry epilogue (tg_rowcoef.cuh) and broadcasts (a, h, lse, s) through
//    a second mbarrier.  Meanwhile the consumers already run phase 1 of the
//    next row on the ring's free slots, so the epilogue is off their path.
//  * Phase 2 re-reads the resident chunks from SMEM and writes
//    dz = p (s + h((z - lse) + H)) - s[v = y] with 128-bit streaming stores,
//    releasing each slot to the producer, which refills it with the next row.
//  * Persistent grid: one CTA per SM (16 warps -> 128 registers / thread),
//    as many clusters as can be co-resident, striding over rows.
#include "tg_common.cuh"
#include "tg_rowcoef.cuh"
#include "tg_vecmath.cuh"

#include <mutex>

namespace tg {

// 14 consumer warps + 1 epilogue warp + 1 producer warp = 16 warps: with the
// 4-warp register allocation granularity this leaves 128 registers per thread
// (17 warps would cap it at 96 and spill).
constexpr int kConsumerWarps = 14;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kEpilogueWarp = kConsumerWarps;
constexpr int kProducerWarp = kConsumerWarps + 1;
constexpr int kFusedThreads = kConsumers + 64;
constexpr int kVecPerThread = 4;                  // 16-byte vectors per consumer thread per chunk
constexpr int kVecPerChunk = kConsumers * kVecPerThread;
constexpr int kChunk = kVecPerChunk * 16;         // 28 KB per TMA bulk copy / ring slot
constexpr int kSlots = 8;                          // ring: 224 KB of the 227 KB opt-in SMEM
constexpr int kMaxPrefixChunks = 8;  // next-row phase-1 chunks run before this row's phase 2
constexpr uint32_t kPrefetchPiece = 65536;  // bytes per L2 prefetch instruction

struct FusedSmemTail {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t xbar[2];   // cluster exchange (DSMEM tx bytes from the peers)
  uint64_t pbar[2];   // consumers -> epilogue warp: per-warp partials written
  uint64_t bbar[2];   // epilogue warp -> consumers: (a, h, lse, s) written
  float4 xdata[2][4];
  float4 wpart[2][kConsumerWarps];
  float4 bcast[2];  // (a, h, lse, s) of a row, from the epilogue warp
  double stats[16];
#ifdef TG_FUSED_PROF
  unsigned long long prof[8];
#endif
};

// ---- optional cycle accounting (profiling build only: -DTG_FUSED_PROF) -------
// prof[0] consumer cycles waiting for ring data (summed over consumer warps)
// prof[1] consumer cycles waiting for the epilogue broadcast (summed over warps)
// prof[2] consumer busy span (warp 0: first wait -> last store)
// prof[3] producer cycles waiting for a free slot
// prof[4] epilogue cycles waiting for the consumer partials
// prof[5] epilogue cycles waiting for the cluster exchange
// prof[6] rows processed by the CTA
#ifdef TG_FUSED_PROF
__device__ unsigned long long g_fused_prof[1024][8];
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

__device__ __forceinline__ void wait_full(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

struct RingBase {
  uint32_t ring, full, empty;  // shared addresses of slot 0's data / full / empty barrier
};

// Ring position as a running chunk counter: slot = c mod kSlots, mbarrier phase
// parity = (c / kSlots) & 1 (kSlots is a power of two, so both are one op).
struct RingIt {
  uint32_t c;
  __device__ __forceinline__ uint32_t slot() const { return c & (kSlots - 1); }
  __device__ __forceinline__ uint32_t phase() const { return (c / kSlots) & 1u; }
  __device__ __forceinline__ uint32_t addr(const RingBase& rb) const { return rb.ring + slot() * kChunk; }
  __device__ __forceinline__ uint32_t full(const RingBase& rb) const { return rb.full + slot() * 8u; }
  __device__ __forceinline__ uint32_t empty(const RingBase& rb) const { return rb.empty + slot() * 8u; }
  __device__ __forceinline__ void next() { ++c; }
  __device__ __forceinline__ void advance(int n) { c += uint32_t(n); }
};

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

// ---- phase 1: one chunk (kVecPerThread vectors per consumer thread) ---------
// kPartial: the chunk may run past the slice end (lanes there use a neutral
// -1e30 vector and skip the sums, but still vote, so the lazy-rescale test is
// always a full-warp vote).  kMaskTail: the chunk holds the tail padding.
template <typename T, bool kPartial, bool kMaskTail>
__device__ __forceinline__ void phase1_chunk(Acc2& acc, RingIt& it, const RingBase& rb,
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
    Pk<T>::clamp(u[g]);
    if (kMaskTail && vec == sl.tail_vec) Pk<T>::mask_from(u[g], sl.tail_valid);
  }
  it.next();
  const float vmax = group_max<T>(u);
  if (__any_sync(0xffffffffu, vmax > acc.m + kSlack)) rescale(acc, vmax);
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g)
    if (!kPartial || valid[g]) accumulate<T>(acc, u[g]);
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
#pragma unroll
  for (int g = 0; g < kVecPerThread; ++g) {
    const int vec = vbase + g * kConsumers + tid;
    if (!kCheck || vec < sl.v1) {
      float d[EPV];
      dz_vec<T, kHasH>(lds128(a + g * kConsumers * 16), d, nl2, av2, hz2);
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
      phase2_chunk<T, kHasH, true>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2, tid);
    else
      phase2_chunk<T, kHasH, false>(it, rb, vbase, sl, dzrow, vy, ye, s_t, nl2, av2, hz2, tid);
    __syncwarp();
    if (lane == 0) arrive_u32(it.empty(rb));
    it.next();
    vbase = vend;
  }
}

// phase 1 over chunks [c0, c1) of a row whose first chunk is at `row_it`
template <typename T>
__device__ __forceinline__ void phase1_range(Acc2& acc, RingIt row_it, const RingBase& rb,
                                             const Slice& sl, int c0, int c1, int tid) {
  RingIt it = row_it;
  it.advance(c0);
  int vbase = sl.v0 + c0 * kVecPerChunk;
  for (int c = c0; c < c1; ++c) {
    const int vend = vbase + kVecPerChunk;
    const bool has_tail = sl.tail_vec >= vbase && sl.tail_vec < vend;
    if (vend <= sl.v1 && !has_tail)
      phase1_chunk<T, false, false>(acc, it, rb, vbase, sl, tid);
    else if (!has_tail)
      phase1_chunk<T, true, false>(acc, it, rb, vbase, sl, tid);
    else
      phase1_chunk<T, true, true>(acc, it, rb, vbase, sl, tid);
    vbase = vend;
  }
}

__device__ __forceinline__ Acc2 acc_init() {
  return Acc2{kNegInf, pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f)};  // nm2 set on first use
}

// waits of the producer / epilogue warps back off with nanosleep so their
// polling does not steal issue slots from the consumer warps on the same SMSP
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(64);
}

template <typename T, int CL>
__global__ void __launch_bounds__(kFusedThreads, 1)
    k_fused_tma(const KParams P, const RowMeta* __restrict__ meta, int prefetch_rows) {
  constexpr int EPV = Vec<T>::N;  // elements per 16-byte vector
  constexpr int ESZ = elem_bytes<T>();
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem;
  FusedSmemTail* tail = reinterpret_cast<FusedSmemTail*>(smem + size_t(kSlots) * kChunk);
  const RingBase rb = {smem_u32(ring), smem_u32(&tail->full[0]), smem_u32(&tail->empty[0])};

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
  sl.nchunk = int((slice_bytes + kChunk - 1) / kChunk);
  sl.tail_vec = (V % EPV) ? nvec - 1 : -1;  // global vector holding columns >= V
  sl.tail_valid = V - (nvec - 1) * EPV;
  // next-row phase-1 chunks that fit in the ring beside this row's slice
  const int pre = min(min(kMaxPrefixChunks, kSlots - sl.nchunk), sl.nchunk);

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], kConsumerWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tail->xbar[i], 1);
      mbar_init(&tail->pbar[i], kConsumerWarps);
      mbar_init(&tail->bbar[i], 1);
    }
    fence_mbar_init();
#ifdef TG_FUSED_PROF
    for (int i = 0; i < 8; ++i) tail->prof[i] = 0ull;
#endif
  }
  if (CL > 1)
    cluster_sync_all();
  else
    __syncthreads();
#ifdef TG_FUSED_PROF
  const long long t_start = clock64();
#endif

  if (warp == kProducerWarp) {
    // ===================== producer warp: bulk TMA into the ring =====================
    if (lane == 0 && sl.nchunk > 0) {
      const uint64_t pol = policy_evict_first();
      const char* base = reinterpret_cast<const char*>(P.logits);
      auto slice_ptr = [&](int64_t row) {
        const int64_t src_row = P.row_index ? P.row_index[row] : row;
        return base + src_row * P.ld * ESZ + int64_t(sl.v0) * 16;
      };
      for (int i = 0; i < prefetch_rows; ++i) {
        const int64_t r = cid + int64_t(i) * ncl;
        if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
      }
      RingIt it = {0u};
      for (int64_t row = cid; row < NR; row += ncl) {
        if (prefetch_rows > 0) {
          const int64_t r = row + int64_t(prefetch_rows) * ncl;
          if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
        }
        const char* src = slice_ptr(row);
        for (int j = 0; j < sl.nchunk; ++j) {
          {
            TG_PROF_T0();
            mbar_wait_u32(it.empty(rb), it.phase() ^ 1u);
            TG_PROF_ADD(tail, 3);
          }
          const uint32_t off = uint32_t(j) * kChunk;
          const uint32_t bytes = min(uint32_t(kChunk), slice_bytes - off);
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
    // ===================== epilogue warp: row reductions + registry epilogue ==========
    // Off the consumers' critical path: while it reduces row k, exchanges with
    // the cluster peers and evaluates the loss terms, the consumers already run
    // phase 1 of row k+1.
    double sd[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) sd[i] = 0.0;
    RingIt pos0 = {0u};
    int64_t k = 0;
    for (int64_t row = cid; row < NR; row += ncl, ++k) {
      const int par = int(k & 1);
      const uint32_t parity = uint32_t((k >> 1) & 1);
      RowMeta cur;
      if (lane == 0) cur = load_meta(meta, row);
      const int y = __ldg(&meta[row].y);
      const int vy = (y >= 0 && y < V) ? (y / EPV) : -1;
      const int ye = (vy >= 0) ? y - vy * EPV : 0;
      {
        TG_PROF_T0();
        mbar_wait_u32(smem_u32(&tail->pbar[par]), parity);
        TG_PROF_ADD(tail, 4);
      }
      const float4 v = (lane < kConsumerWarps) ? tail->wpart[par][lane]
                                               : make_float4(kNegInf, 0.f, 0.f, 0.f);
      const Online cta = warp_merge(Online{v.x, v.y, v.z});
      // the target logit, read straight from the still-resident chunk (raw, unclamped)
      float czy = kNegInf;
      if (vy >= sl.v0 && vy < sl.v1) {
        const int off = vy - sl.v0;
        RingIt at = pos0;
        at.advance(off / kVecPerChunk);
        czy = Pk<T>::elem(lds128(at.addr(rb) + uint32_t(off % kVecPerChunk) * 16), ye);
      }
      Online tot = cta;
      float tzy = czy;
      if constexpr (CL > 1) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&tail->xbar[par], (CL - 1) * 16);
          const uint32_t my_slot = smem_u32(&tail->xdata[par][rank]);
          const uint32_t bar = smem_u32(&tail->xbar[par]);
#pragma unroll
          for (int r = 0; r < CL; ++r) {
            if (r == int(rank)) continue;
            st_async_v4(map_to_rank(my_slot, r), cta.m, cta.s, cta.t, czy, map_to_rank(bar, r));
          }
        }
        {
          TG_PROF_T0();
          mbar_wait_cluster(&tail->xbar[par], parity);
          TG_PROF_ADD(tail, 5);
        }
        tot = {kNegInf, 0.f, 0.f};
        tzy = kNegInf;
#pragma unroll
        for (int r = 0; r < CL; ++r) {  // fixed rank order: identical result on every CTA
          const float4 w = (r == int(rank)) ? make_float4(cta.m, cta.s, cta.t, czy)
                                            : tail->xdata[par][r];
          tot = online_merge(tot, Online{w.x, w.y, w.z});
          tzy = fmaxf(tzy, w.w);
        }
      }
      if (lane == 0) {
        const float lse = tot.m + logf(tot.s);
        const float H = lse - tot.t / tot.s;
        const bool bad_target = (cur.flags & 2u) != 0;
        const float lp = tzy - lse;
        RowTerms o = meta_terms(P, cur, lp, H);
        if (bad_target) {
          o.s = 0.f;
          o.h = 0.f;
        }
        tail->bcast[par] = make_float4(o.s + o.h * (H - lse), o.h, lse, o.s);
        arrive_u32(smem_u32(&tail->bbar[par]));
        if (rank == 0) {  // outputs + statistics, after the broadcast
          P.lp[row] = lp;
          P.ent[row] = H;
          P.lse[row] = lse;
          const bool nonfin = !(finite_f(lse) && finite_f(lp) && finite_f(H) && finite_f(o.s) &&
                                finite_f(o.h));
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
      pos0.advance(sl.nchunk);
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
    }
  } else {
    // ===================== consumer warps =====================
    RingIt pos0 = {0u};  // the current row's first chunk
    Acc2 acc = acc_init();
    if (cid < NR) phase1_range<T>(acc, pos0, rb, sl, 0, pre, tid);  // first row's prefix
    int y_cur = (cid < NR) ? __ldg(&meta[cid].y) : 0;
    int64_t k = 0;
    for (int64_t row = cid; row < NR; row += ncl, ++k) {
      const int64_t nrow = row + ncl;
      const int y_next = (nrow < NR) ? __ldg(&meta[nrow].y) : 0;  // prefetch
      const int y = y_cur;
      const int vy = (y >= 0 && y < V) ? (y / EPV) : -1;  // global vector holding the target
      const int ye = (vy >= 0) ? y - vy * EPV : 0;
      const int par = int(k & 1);

      // ---------------- phase 1 (rest of the row) ----------------
      phase1_range<T>(acc, pos0, rb, sl, pre, sl.nchunk, tid);
      Online o;
      {
        float s0, s1, t0, t1;
        upk2(acc.s2, s0, s1);
        upk2(acc.t2, t0, t1);
        o = warp_merge(Online{acc.m, s0 + s1, t0 + t1});
      }
      if (lane == 0) {
        tail->wpart[par][warp] = make_float4(o.m, o.s, o.t, 0.f);
        arrive_u32(smem_u32(&tail->pbar[par]));
      }
      // ---------------- phase 1 prefix of the next row (hides the epilogue) ----------
      RingIt npos = pos0;
      npos.advance(sl.nchunk);
      acc = acc_init();
      if (nrow < NR) phase1_range<T>(acc, npos, rb, sl, 0, pre, tid);

      // ---------------- phase 2: dz from the resident slice ----------------
      {
        TG_PROF_T0();
        mbar_wait_u32(smem_u32(&tail->bbar[par]), uint32_t((k >> 1) & 1));
        TG_PROF_ADD(tail, 1);
      }
      const float4 bc = tail->bcast[par];
      const float a = bc.x, hz = bc.y, s_t = bc.w;
      const float lseL = bc.z * kLog2e;
      const uint64_t nl2 = pk2(-lseL, -lseL), av2 = pk2(a, a), hz2 = pk2(hz, hz);
      char* dzrow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
      if (hz == 0.f)
        phase2_row<T, false>(sl, pos0, rb, dzrow, vy, ye, s_t, nl2, av2, hz2, tid, lane);
      else
        phase2_row<T, true>(sl, pos0, rb, dzrow, vy, ye, s_t, nl2, av2, hz2, tid, lane);
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
#ifdef TG_FUSED_PROF
  __syncthreads();
  if (tid < 8) g_fused_prof[blockIdx.x][tid] = tail->prof[tid];
#endif
}

// ---------------------------------------------------------------------------
// host-side launch helper (called from tg_api.cu)

size_t fused_smem_bytes(int n_slots) { return size_t(n_slots) * kChunk + sizeof(FusedSmemTail); }

template <typename T, int CL>
static cudaError_t launch_fused_t(const KParams& P, const RowMeta* meta, int n_ctas,
                                  int prefetch_rows, cudaStream_t stream) {
  const size_t smem = fused_smem_bytes(kSlots);
  cudaError_t e = cudaFuncSetAttribute(k_fused_tma<T, CL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_fused_tma<T, CL>, P, meta, prefetch_rows);
}

cudaError_t launch_fused(const KParams& P, const void* meta, int cl, int n_slots, int n_ctas,
                         int prefetch_rows, cudaStream_t stream) {
  if (n_slots != kSlots) return cudaErrorInvalidValue;
  const RowMeta* m = reinterpret_cast<const RowMeta*>(meta);
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
  return int(cudaMemcpyFromSymbol(out, g_fused_prof, size_t(n_ctas) * 8 * sizeof(unsigned long long)));
}
#endif

int fused_chunk_bytes() { return kChunk; }
int fused_max_slots() { return kSlots; }
size_t rowmeta_bytes() { return sizeof(RowMeta); }

}  // namespace tg
