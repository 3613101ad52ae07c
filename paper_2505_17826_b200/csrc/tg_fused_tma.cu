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
//    (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first), in CHUNK-byte
//    pieces with one full / empty mbarrier pair per ring slot.
//  * 16 consumer warps run phase 1 on each chunk as it lands (online max /
//    sum-exp / sum p*z and the target logit), reduce across warps (one named
//    barrier), then across the cluster through DSMEM (st.async into each
//    peer's exchange slot, completing tx bytes on the peer's mbarrier; every
//    CTA merges the CL partials in rank order so all CTAs get bit-identical
//    lse / H).
//  * The per-row epilogue (tg_rowcoef.cuh) turns (lp, H) into (s, h); phase 2
//    re-reads the chunks from SMEM, writes dz = p (s + h((z - lse) + H)) - s[v=y]
//    with 128-bit streaming stores, and releases each slot to the producer,
//    which is already loading the next row into the freed space (the ring is
//    larger than one row slice, so HBM reads never drain).
//  * Persistent grid: one CTA per SM, clusters stride over rows.
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
constexpr int kVecPerChunk = kChunk / 16;

struct FusedSmemTail {
  uint64_t full[kMaxSlots];
  uint64_t empty[kMaxSlots];
  uint64_t xbar[2];
  float4 xdata[2][4];
  float4 wpart[2][kConsumerWarps];
};

template <typename T, int CL>
__global__ void __launch_bounds__(kFusedThreads, 1)
    k_fused_tma(const KParams P, const RowMeta* __restrict__ meta, int n_slots) {
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
  const int64_t NR = P.n_rows, V = P.vocab;

  // column slice of this CTA, in 16-byte vectors
  const int64_t nvec = (V + EPV - 1) / EPV;
  const int64_t v0 = (int64_t(rank) * nvec) / CL;
  const int64_t v1 = (int64_t(rank + 1) * nvec) / CL;
  const uint32_t slice_bytes = uint32_t((v1 - v0) * 16);
  const int nchunk = int((slice_bytes + kChunk - 1) / kChunk);

  if (tid == 0) {
    for (int i = 0; i < n_slots; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], kConsumerWarps);
    }
    mbar_init(&tail->xbar[0], 1);
    mbar_init(&tail->xbar[1], 1);
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
      int slot = 0;
      uint32_t phase = 0;
      for (int64_t row = cid; row < NR; row += ncl) {
        const int64_t src_row = P.row_index ? P.row_index[row] : row;
        const char* src = base + src_row * P.ld * ESZ + v0 * 16;
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
    RowStats st;
    st.zero();
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
      const int64_t y = cur.y;
      const int64_t vy = (y >= 0 && y < V) ? (y / EPV) : -1;  // global vector holding the target

      // ---------------- phase 1: online max / sum-exp / sum p*z ----------------
      Online acc = {kNegInf, 0.f, 0.f};
      float zy = kNegInf;
      {
        int slot = slot0;
        uint32_t phase = phase0;
        for (int j = 0; j < nchunk; ++j) {
          mbar_wait(&tail->full[slot], phase);
          const uint4* cv = reinterpret_cast<const uint4*>(ring + size_t(slot) * kChunk);
          const int64_t vbase = v0 + int64_t(j) * kVecPerChunk;
          const int nv = int(min(int64_t(kVecPerChunk), v1 - vbase));
          for (int q = tid; q < nv; q += kConsumers) {
            float x[EPV];
            Vec<T>::unpack(cv[q], x);
            const int64_t vec = vbase + q;
            const int64_t col0 = vec * EPV;
            if (col0 + EPV > V) {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (col0 + e >= V) x[e] = kNegInf;
            }
            if (vec == vy) {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (col0 + e == y) zy = x[e];
            }
            float vmax = x[0];
#pragma unroll
            for (int e = 1; e < EPV; ++e) vmax = fmaxf(vmax, x[e]);
            if (vmax > acc.m) {
              const float sc = ex2((acc.m - vmax) * kLog2e);
              acc.s *= sc;
              acc.t *= sc;
              acc.m = vmax;
            }
            if (acc.m != kNegInf) {
              const float mL = acc.m * kLog2e;
#pragma unroll
              for (int e = 0; e < EPV; ++e) {
                const float xc = fmaxf(x[e], kClampLow);
                const float p = ex2(fmaf(xc, kLog2e, -mL));
                acc.s += p;
                acc.t = fmaf(p, xc, acc.t);
              }
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
        st.add(o, lp, H, bad_target, nonfin);
      }
      // ---------------- phase 2: dz from the resident slice ----------------
      const float a = o.s + o.h * (H - lse);
      const float hz = o.h;
      const float lseL = lse * kLog2e;
      const float s_t = o.s;
      char* dzrow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
      {
        int slot = slot0;
        uint32_t phase = phase0;
        for (int j = 0; j < nchunk; ++j) {
          const uint4* cv = reinterpret_cast<const uint4*>(ring + size_t(slot) * kChunk);
          const int64_t vbase = v0 + int64_t(j) * kVecPerChunk;
          const int nv = int(min(int64_t(kVecPerChunk), v1 - vbase));
          for (int q = tid; q < nv; q += kConsumers) {
            float x[EPV];
            Vec<T>::unpack(cv[q], x);
            const int64_t vec = vbase + q;
            const int64_t col0 = vec * EPV;
            float d[EPV];
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              const float xc = fmaxf(x[e], kClampLow);
              const float p = ex2(fmaf(xc, kLog2e, -lseL));
              d[e] = p * fmaf(hz, xc, a);
            }
            if (vec == vy) {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (col0 + e == y) d[e] -= s_t;
            }
            if (col0 + EPV <= V) {
              st_stream(dzrow + vec * 16, Vec<T>::pack(d));
            } else {
#pragma unroll
              for (int e = 0; e < EPV; ++e)
                if (col0 + e < V) Vec<T>::store1(P.dz, row * P.ld_out + col0 + e, d[e]);
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
    if (tid == 0) st.store(P.partials + size_t(blockIdx.x) * TG_NSTAT);
  }
  if (CL > 1)
    cluster_sync_all();  // no CTA leaves while a peer may still st.async into it
}

// ---------------------------------------------------------------------------
// host-side launch helper (called from tg_api.cu)

size_t fused_smem_bytes(int n_slots) { return size_t(n_slots) * kChunk + sizeof(FusedSmemTail); }

template <typename T, int CL>
static cudaError_t launch_fused_t(const KParams& P, const RowMeta* meta, int n_slots, int n_ctas,
                                  cudaStream_t stream) {
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
  return cudaLaunchKernelEx(&cfg, k_fused_tma<T, CL>, P, meta, n_slots);
}

cudaError_t launch_fused(const KParams& P, const void* meta, int cl, int n_slots, int n_ctas,
                         cudaStream_t stream) {
  const RowMeta* m = reinterpret_cast<const RowMeta*>(meta);
  if (P.dtype == TG_DTYPE_BF16) {
    if (cl == 1) return launch_fused_t<bf16_t, 1>(P, m, n_slots, n_ctas, stream);
    if (cl == 2) return launch_fused_t<bf16_t, 2>(P, m, n_slots, n_ctas, stream);
    if (cl == 4) return launch_fused_t<bf16_t, 4>(P, m, n_slots, n_ctas, stream);
  } else {
    if (cl == 1) return launch_fused_t<float, 1>(P, m, n_slots, n_ctas, stream);
    if (cl == 2) return launch_fused_t<float, 2>(P, m, n_slots, n_ctas, stream);
    if (cl == 4) return launch_fused_t<float, 4>(P, m, n_slots, n_ctas, stream);
  }
  return cudaErrorInvalidValue;
}

int fused_chunk_bytes() { return kChunk; }
int fused_max_slots() { return kMaxSlots; }
size_t rowmeta_bytes() { return sizeof(RowMeta); }

}  // namespace tg
