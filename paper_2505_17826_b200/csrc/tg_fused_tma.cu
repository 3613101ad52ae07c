// tg_fused_tma.cu -- K1: fused single-pass logprob + loss + dlogits over [T, V] logits.
//
// Replaces, per trainable row, policy.logprob (policy.py:194-212),
// policy.grad_logprob (policy.py:253-270) and the per-variant axpy of the
// loss's coefficient (algorithms.py:240-242, 263-266) -- plus the north_star
// PPO clip / KL / entropy terms -- with one read of the row from HBM and one
// write of d loss / d logits (4V bytes per row, the HBM roofline minimum).
//
// Design (B200-first):
//  * A thread-block cluster of CL CTAs (CL = 1 for V <= ~100k bf16, 2 for
//    Qwen's 151,936) owns one row at a time; CTA rank r owns a contiguous
//    column slice of the row.  The slice never leaves the SM: a producer warp
//    streams it into a shared-memory ring with 1-D bulk TMA
//    (cp.async.bulk ... mbarrier::complete_tx), one chunk per ring slot with
//    a full / empty mbarrier pair, and keeps HBM busy across row boundaries
//    by prefetching upcoming rows' slices into L2 (cp.async.bulk.prefetch.L2)
//    -- the ring holds ~1.5 slices, L2 holds the look-ahead.
//  * 15 consumer warps (one 16-byte vector per thread per chunk) run phase 1
//    on each chunk as it lands: online max / sum-exp / sum p*z and the target
//    logit; -inf logits are clamped to -1e30 with packed bf16x2 max so no
//    per-element guard is needed.  One named barrier reduces across warps;
//    DSMEM (st.async into each peer's exchange slot, completing tx bytes on
//    the peer's mbarrier) reduces across the cluster.  Every CTA merges the
//    CL partials in rank order, so all CTAs get bit-identical lse / H.
//  * The per-row epilogue (tg_rowcoef.cuh) turns (lp, H) into (s, h); phase 2
//    re-reads the chunks from SMEM, writes dz = p (s + h((z - lse) + H)) - s[v=y]
//    with 128-bit streaming stores and releases each slot to the producer.
//  * Persistent grid: one CTA per SM (16 warps -> 128 registers / thread),
//    clusters stride over rows.
#include "tg_common.cuh"
#include "tg_rowcoef.cuh"

namespace tg {

// 15 consumer warps + 1 producer warp = 16 warps: with the 4-warp register
// allocation granularity this leaves 128 registers per thread (17 warps would
// cap it at 96 and spill).  One 16-byte vector per consumer thread per chunk.
constexpr int kConsumerWarps = 15;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kFusedThreads = kConsumers + 32;
constexpr int kChunk = kConsumers * 16;  // 7680 bytes per TMA bulk copy / ring slot
constexpr int kMaxSlots = 30;
constexpr uint32_t kPrefetchPiece = 65536;  // bytes per L2 prefetch instruction

struct FusedSmemTail {
  uint64_t full[kMaxSlots];
  uint64_t empty[kMaxSlots];
  uint64_t xbar[2];
  float4 xdata[2][4];
  float4 wpart[2][kConsumerWarps];
  double stats[16];
};

// ---- packed-element helpers (bf16: 8 per vector, fp32: 4 per vector) --------

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

constexpr uint32_t kBf16NegBig2 = 0xF149F149u;  // (-1.0e30, -1.0e30) as bf16x2
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
  __device__ __forceinline__ static float vmax(const uint4& u) {
    const uint32_t m = bmax2(bmax2(u.x, u.y), bmax2(u.z, u.w));
    return fmaxf(__uint_as_float(m << 16), __uint_as_float(m & 0xffff0000u));
  }
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
  __device__ __forceinline__ static float vmax(const uint4& u) {
    return fmaxf(fmaxf(__uint_as_float(u.x), __uint_as_float(u.y)),
                 fmaxf(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  __device__ __forceinline__ static void mask_from(uint4& u, int n) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e >= n) w[e] = __float_as_uint(kNegBig);
  }
  __device__ __forceinline__ static float elem(const uint4& u, int e) {
    return __uint_as_float(e == 0 ? u.x : e == 1 ? u.y : e == 2 ? u.z : u.w);
  }
};

__device__ __forceinline__ void prefetch_l2(const char* p, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += kPrefetchPiece) {
    const uint32_t n = min(kPrefetchPiece, bytes - off);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(n) : "memory");
  }
}

template <typename T, int CL>
__global__ void __launch_bounds__(kFusedThreads, 1)
    k_fused_tma(const KParams P, const RowMeta* __restrict__ meta, int n_slots,
                int prefetch_rows) {
  constexpr int EPV = Vec<T>::N;  // elements per 16-byte vector
  constexpr int ESZ = elem_bytes<T>();
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem;
  FusedSmemTail* tail = reinterpret_cast<FusedSmemTail*>(smem + size_t(n_slots) * kChunk);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = (CL > 1) ? cluster_ctarank() : 0u;
  const int64_t cid = (CL > 1) ? int64_t(cluster_id_x()) : int64_t(blockIdx.x);
  const int64_t ncl = (CL > 1) ? int64_t(n_clusters_x()) : int64_t(gridDim.x);
  const int64_t NR = P.n_rows;
  const int V = int(P.vocab);

  // column slice of this CTA, in 16-byte vectors (32-bit: V < 2^31)
  const int nvec = (V + EPV - 1) / EPV;
  const int v0 = int((int64_t(rank) * nvec) / CL);
  const int v1 = int((int64_t(rank + 1) * nvec) / CL);
  const uint32_t slice_bytes = uint32_t(v1 - v0) * 16u;
  const int nchunk = int((slice_bytes + kChunk - 1) / kChunk);
  const int tail_vec = (V % EPV) ? nvec - 1 : -1;  // global vector holding columns >= V
  const int tail_valid = V - (nvec - 1) * EPV;

  if (tid == 0) {
    for (int i = 0; i < n_slots; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], kConsumerWarps);
    }
    mbar_init(&tail->xbar[0], 1);
    mbar_init(&tail->xbar[1], 1);
    for (int i = 0; i < 16; ++i) tail->stats[i] = 0.0;
    fence_mbar_init();
  }
  if (CL > 1)
    cluster_sync_all();
  else
    __syncthreads();

  if (warp == kConsumerWarps) {
    // ===================== producer warp: bulk TMA into the ring =====================
    if (lane == 0 && nchunk > 0) {
      const uint64_t pol = policy_evict_first();
      const char* base = reinterpret_cast<const char*>(P.logits);
      auto slice_ptr = [&](int64_t row) {
        const int64_t src_row = P.row_index ? P.row_index[row] : row;
        return base + src_row * P.ld * ESZ + int64_t(v0) * 16;
      };
      for (int i = 0; i < prefetch_rows; ++i) {
        const int64_t r = cid + int64_t(i) * ncl;
        if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
      }
      int slot = 0;
      uint32_t phase = 0;
      for (int64_t row = cid; row < NR; row += ncl) {
        if (prefetch_rows > 0) {
          const int64_t r = row + int64_t(prefetch_rows) * ncl;
          if (r < NR) prefetch_l2(slice_ptr(r), slice_bytes);
        }
        const char* src = slice_ptr(row);
        for (int j = 0; j < nchunk; ++j) {
          mbar_wait(&tail->empty[slot], phase ^ 1u);
          const uint32_t off = uint32_t(j) * kChunk;
          const uint32_t bytes = min(uint32_t(kChunk), slice_bytes - off);
          mbar_arrive_expect_tx(&tail->full[slot], bytes);
          tma_load_1d(ring + size_t(slot) * kChunk, src + off, bytes, &tail->full[slot], pol);
          if (++slot == n_slots) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== consumer warps =====================
    const bool writer = (rank == 0) && (tid == 0);
    int slot0 = 0;  // ring slot of the current row's first chunk
    uint32_t phase0 = 0;
    int64_t k = 0;
    RowMeta cur;
    if (cid < NR) cur = load_meta(meta, cid);
    for (int64_t row = cid; row < NR; row += ncl, ++k) {
      const int64_t nrow = row + ncl;
      RowMeta nxt = cur;
      if (nrow < NR) nxt = load_meta(meta, nrow);  // prefetch next row's metadata
      const int y = cur.y;
      const int vy = (y >= 0 && y < V) ? (y / EPV) : -1;  // global vector holding the target
      const int ye = (vy >= 0) ? y - vy * EPV : 0;

      // ---------------- phase 1: online max / sum-exp / sum p*z ----------------
      Online acc = {kNegInf, 0.f, 0.f};
      float zy = kNegInf;
      {
        int slot = slot0;
        uint32_t phase = phase0;
        int vbase = v0;
        for (int j = 0; j < nchunk; ++j, vbase += kConsumers) {
          const int nv = min(kConsumers, v1 - vbase);
          mbar_wait(&tail->full[slot], phase);
          if (tid < nv) {
            uint4 u = reinterpret_cast<const uint4*>(ring + size_t(slot) * kChunk)[tid];
            Pk<T>::clamp(u);
            const int vec = vbase + tid;
            if (vec == tail_vec) Pk<T>::mask_from(u, tail_valid);
            if (vec == vy) zy = Pk<T>::elem(u, ye);
            const float vmax = Pk<T>::vmax(u);
            if (vmax > acc.m) {
              const float sc = ex2((acc.m - vmax) * kLog2e);
              acc.s *= sc;
              acc.t *= sc;
              acc.m = vmax;
            }
            float x[EPV];
            Vec<T>::unpack(u, x);
            const float mL = acc.m * kLog2e;
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              const float p = ex2(fmaf(x[e], kLog2e, -mL));
              acc.s += p;
              acc.t = fmaf(p, x[e], acc.t);
            }
          }
          if (++slot == n_slots) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
      // ---------------- reductions: warp -> CTA -> cluster ----------------
      acc = warp_merge(acc);
      zy = warp_max(zy);
      const int par = int(k & 1);
      if (lane == 0) tail->wpart[par][warp] = make_float4(acc.m, acc.s, acc.t, zy);
      named_bar_sync(1, kConsumers);
      Online cta = {kNegInf, 0.f, 0.f};
      float czy = kNegInf;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float4 v = tail->wpart[par][w];
        cta = online_merge(cta, Online{v.x, v.y, v.z});
        czy = fmaxf(czy, v.w);
      }
      Online tot = cta;
      float tzy = czy;
      if constexpr (CL > 1) {
        if (tid == 0) {
          mbar_arrive_expect_tx(&tail->xbar[par], (CL - 1) * 16);
          const uint32_t my_slot = smem_u32(&tail->xdata[par][rank]);
          const uint32_t bar = smem_u32(&tail->xbar[par]);
#pragma unroll
          for (int r = 0; r < CL; ++r) {
            if (r == int(rank)) continue;
            st_async_v4(map_to_rank(my_slot, r), cta.m, cta.s, cta.t, czy, map_to_rank(bar, r));
          }
        }
        mbar_wait_cluster(&tail->xbar[par], uint32_t((k >> 1) & 1));
        tot = {kNegInf, 0.f, 0.f};
        tzy = kNegInf;
#pragma unroll
        for (int r = 0; r < CL; ++r) {  // fixed rank order: identical result on every CTA
          float4 v = (r == int(rank)) ? make_float4(cta.m, cta.s, cta.t, czy)
                                      : tail->xdata[par][r];
          tot = online_merge(tot, Online{v.x, v.y, v.z});
          tzy = fmaxf(tzy, v.w);
        }
      }
      const float lse = tot.m + logf(tot.s);
      const float H = lse - tot.t / tot.s;
      const bool bad_target = (cur.flags & 2u) != 0;
      const float lp = tzy - lse;
      RowTerms o = meta_terms(P, cur, lp, H);
      if (bad_target) {
        o.s = 0.f;
        o.h = 0.f;
      }
      if (writer) {
        P.lp[row] = lp;
        P.ent[row] = H;
        P.lse[row] = lse;
        const bool nonfin = !(finite_f(lse) && finite_f(lp) && finite_f(H) && finite_f(o.s) &&
                              finite_f(o.h));
        double* sd = tail->stats;
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
      // ---------------- phase 2: dz from the resident slice ----------------
      const float hz = o.h;
      const float a = o.s + hz * (H - lse);
      const float lseL = lse * kLog2e;
      const float s_t = o.s;
      char* dzrow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
      {
        int slot = slot0;
        uint32_t phase = phase0;
        int vbase = v0;
        for (int j = 0; j < nchunk; ++j, vbase += kConsumers) {
          const int nv = min(kConsumers, v1 - vbase);
          if (tid < nv) {
            uint4 u = reinterpret_cast<const uint4*>(ring + size_t(slot) * kChunk)[tid];
            Pk<T>::clamp(u);
            float x[EPV], d[EPV];
            Vec<T>::unpack(u, x);
            if (hz == 0.f) {
#pragma unroll
              for (int e = 0; e < EPV; ++e) d[e] = ex2(fmaf(x[e], kLog2e, -lseL)) * a;
            } else {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                d[e] = ex2(fmaf(x[e], kLog2e, -lseL)) * fmaf(hz, x[e], a);
            }
            const int vec = vbase + tid;
            if (vec == vy) {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (e == ye) d[e] -= s_t;
            }
            if (vec != tail_vec) {
              st_stream(dzrow + int64_t(vec) * 16, Vec<T>::pack(d));
            } else {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (e < tail_valid) Vec<T>::store1(dzrow, int64_t(vec) * EPV + e, d[e]);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&tail->empty[slot]);
          if (++slot == n_slots) {
            slot = 0;
            phase ^= 1u;
          }
        }
        slot0 = slot;
        phase0 = phase;
      }
      cur = nxt;
    }
    // rank 0 of each cluster accumulated its rows; other ranks store zeros
    if (tid == 0) {
      const double* sd = tail->stats;
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
  }
  if (CL > 1)
    cluster_sync_all();  // no CTA leaves while a peer may still st.async into it
}

// ---------------------------------------------------------------------------
// host-side launch helper (called from tg_api.cu)

size_t fused_smem_bytes(int n_slots) { return size_t(n_slots) * kChunk + sizeof(FusedSmemTail); }

template <typename T, int CL>
static cudaError_t launch_fused_t(const KParams& P, const RowMeta* meta, int n_slots, int n_ctas,
                                  int prefetch_rows, cudaStream_t stream) {
  const size_t smem = fused_smem_bytes(n_slots);
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
  return cudaLaunchKernelEx(&cfg, k_fused_tma<T, CL>, P, meta, n_slots, prefetch_rows);
}

cudaError_t launch_fused(const KParams& P, const void* meta, int cl, int n_slots, int n_ctas,
                         int prefetch_rows, cudaStream_t stream) {
  const RowMeta* m = reinterpret_cast<const RowMeta*>(meta);
  if (P.dtype == TG_DTYPE_BF16) {
    if (cl == 1) return launch_fused_t<bf16_t, 1>(P, m, n_slots, n_ctas, prefetch_rows, stream);
    if (cl == 2) return launch_fused_t<bf16_t, 2>(P, m, n_slots, n_ctas, prefetch_rows, stream);
    if (cl == 4) return launch_fused_t<bf16_t, 4>(P, m, n_slots, n_ctas, prefetch_rows, stream);
  } else {
    if (cl == 1) return launch_fused_t<float, 1>(P, m, n_slots, n_ctas, prefetch_rows, stream);
    if (cl == 2) return launch_fused_t<float, 2>(P, m, n_slots, n_ctas, prefetch_rows, stream);
    if (cl == 4) return launch_fused_t<float, 4>(P, m, n_slots, n_ctas, prefetch_rows, stream);
  }
  return cudaErrorInvalidValue;
}

int fused_chunk_bytes() { return kChunk; }
int fused_max_slots() { return kMaxSlots; }
size_t rowmeta_bytes() { return sizeof(RowMeta); }

}  // namespace tg
