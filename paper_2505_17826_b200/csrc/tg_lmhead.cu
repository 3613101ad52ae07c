// tg_lmhead.cu -- K7: fused LM-head + log-softmax forward on the 5th-gen tensor cores.
//
// the logits "producer".  For hidden states X [T, d] and the
// LM-head W [V, d] (both bf16, K-contiguous) it computes per row
//     lse_t = log sum_v exp(z_tv),  lp_t = z_{t,y_t} - lse_t,  H_t = lse_t - sum_v p_tv z_tv
// with z = X W^T, without ever writing the [T, V] logits to HBM: the logits of a
// 128 x 256 tile live only in TMEM and are folded into per-row online
// (max, sum e, sum e z) state by the epilogue warps.  This is the forward-only
// logprob service of §8(f-3) (policy.logprob, policy.py:194-212, for old / ref
// logprob recompute) moved in front of the GEMM.
//
// Design (sm_100a, one CTA per SM, persistent over 128-row blocks):
//  * warp 0, one lane: TMA producer.  For every (row block, vocab tile, k-block)
//    it loads the X tile [128 x 64] and the W tile [256 x 64] (128-byte swizzle)
//    into a 4-stage shared-memory ring (48 KB per stage), full / empty mbarriers.
//  * warp 1, one lane: MMA issuer.  tcgen05.mma.cta_group::1.kind::f16
//    (M = 128, N = 256, K = 16, bf16 x bf16 -> fp32) into one of two TMEM
//    accumulators (2 x 256 columns); tcgen05.commit frees ring slots and
//    signals the epilogue when a tile's accumulation is complete.
//  * warp 2: TMEM allocation / deallocation (512 columns).
//  * warps 4..7: epilogue.  Warp q reads TMEM lanes [32q, 32q + 32) (row = lane)
//    with tcgen05.ld.32x32b.x32, updates its row's online state in packed fp32x2
//    arithmetic, gathers the target logit, and hands the accumulator back; the
//    next tile's MMAs already run into the other accumulator.
//  Rows past T and vocabulary columns past V come in as TMA zero fill and are
//  masked in the epilogue.
//
// Backward (kDz = true, tg_lmhead_dlogits): the same pipeline over one
// vocabulary chunk; the epilogue writes bf16 d loss / d z = p (a + hz z) - s [v = y]
// of each tile (policy.grad_logprob, policy.py:253-270, behind an LM head)
// through swizzled shared-memory staging and TMA bulk-tensor stores.  2-CTA
// pairs by default for this mode (see lm_pair_mode).
#include "tg_common.cuh"
#include "tg_umma.cuh"
#include "tg_vecmath.cuh"

namespace tg {

constexpr int LM_BM = 128;                       // rows per tile (UMMA M)
constexpr int LM_BN = 256;                       // vocabulary columns per tile (UMMA N)
constexpr int LM_BK = 64;                        // K per stage: 64 bf16 = one 128-byte swizzle row
constexpr int LM_UK = 16;                        // K per tcgen05.mma (kind::f16)
constexpr int LM_STAGES = 4;
constexpr int LM_A_BYTES = LM_BM * LM_BK * 2;    // 16 KB
constexpr int LM_B_BYTES = LM_BN * LM_BK * 2;    // 32 KB
constexpr int LM_STAGE_BYTES = LM_A_BYTES + LM_B_BYTES;
constexpr int LM_THREADS = 256;                  // 8 warps
constexpr int LM_EPI_WARP0 = 4;
constexpr uint32_t LM_TMEM_COLS = 512;           // 2 accumulators x 256 fp32 columns

struct LmParams {
  int64_t n_rows, vocab, dim;
  int64_t col0, n_cols;   // vocabulary columns [col0, col0 + n_cols) covered by the tiles
  int n_split;            // vocabulary splits per row block (> 1: partials + merge kernel)
  int sp_major;           // work-unit order: split-major (1) or row-block-major (0)
  float4* partial;        // [n_split, T] (m, sum e, sum e z, z_target) when n_split > 1
  const int32_t* target;  // [T] (may be null: lp not produced)
  float* lp;              // [T]
  float* ent;             // [T]
  float* lse;             // [T]
  // backward (kDz): dz[t, j] = p (a + hz z) - s [col0 + j == y] for the chunk
  const float* coef;      // [3, T]: a, hz, s
  const float* lse_in;    // [T]
  uint16_t* dz;           // bf16 [T, ld_dz]
  int64_t ld_dz;
};

constexpr int LM_MAX_STAGES = 6;

struct LmSmemTail {
  uint64_t full[LM_MAX_STAGES];
  uint64_t empty[LM_MAX_STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

// per-CTA stage: X tile 16 KB + W tile 32 KB (single) or 16 KB (pair: half of it);
// the pair variant affords 6 stages in the same shared memory
template <bool kPair>
constexpr int lm_stages() { return kPair ? 6 : LM_STAGES; }
template <bool kPair>
constexpr int lm_stage_bytes() { return LM_A_BYTES + (kPair ? LM_BN / 2 : LM_BN) * LM_BK * 2; }
// backward epilogue staging: per epilogue warp two [32 rows x 32 bf16] tiles
// (64-byte rows, 64-byte swizzle) that a TMA bulk-tensor store writes out
constexpr int LM_DZ_TILE_BYTES = 32 * 64;
constexpr int LM_DZ_STAGE_BYTES = 4 * 2 * LM_DZ_TILE_BYTES;  // 16 KB
template <bool kPair>
size_t lm_smem_bytes() {
  return size_t(lm_stages<kPair>()) * lm_stage_bytes<kPair>() + LM_DZ_STAGE_BYTES +
         sizeof(LmSmemTail) + 1024;
}

// ---- PTX wrappers -------------------------------------------------------------

// TMA bulk-tensor store of a shared-memory tile (bulk-group completion)
__device__ __forceinline__ void lm_tma_store_2d(const CUtensorMap* map, uint32_t src, int c0,
                                                int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
// wait until at most N committed stores still read shared memory
template <int N>
__device__ __forceinline__ void lm_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <bool kPair>
constexpr uint32_t lm_idesc_t() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(LM_BN >> 3) << 17) |
         (uint32_t((kPair ? 2 * LM_BM : LM_BM) >> 4) << 24);
}

// ---- the kernel -----------------------------------------------------------------
// kPair = false: one CTA per 128-row block, tcgen05.mma.cta_group::1 (M 128, N 256).
// kPair = true : a 2-CTA cluster per 256-row block; each CTA stages its own 128 X
//   rows and half of the 256-row W tile, the leader (rank 0) issues
//   tcgen05.mma.cta_group::2 (M 256, N 256) reading both CTAs' shared memory, and
//   each CTA's TMEM receives its 128 rows: per SM the W-tile traffic halves.

// kDz = false: the forward (per-row lse / entropy / lp).  kDz = true: the
// backward of one vocabulary chunk -- the epilogue turns each logit tile into
// bf16 d loss / d z from the forward's lse and the loss's row coefficients.
template <bool kPair, bool kDz>
__global__ void __launch_bounds__(LM_THREADS, 1)
    k_lmhead_logprob(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmD, const LmParams P) {
  constexpr int B_ROWS = kPair ? LM_BN / 2 : LM_BN;      // W rows staged per CTA
  constexpr int STAGE = lm_stage_bytes<kPair>();
  constexpr int NST = lm_stages<kPair>();
  constexpr int ROWS_PER_UNIT = kPair ? 2 * LM_BM : LM_BM;
  extern __shared__ __align__(1024) unsigned char lm_smem_raw[];
  // 1 KB alignment for the 128-byte swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(lm_smem_raw) + 1023) & ~uintptr_t(1023));
  LmSmemTail* tail =
      reinterpret_cast<LmSmemTail*>(smem + size_t(NST) * STAGE + LM_DZ_STAGE_BYTES);
  const uint32_t ring = smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit0 = kPair ? int(cluster_id_x()) : int(blockIdx.x);
  const int unit_stride = kPair ? int(n_clusters_x()) : int(gridDim.x);
  const int64_t T = P.n_rows;
  const int V = int(P.vocab);
  const int n_mb = int((T + ROWS_PER_UNIT - 1) / ROWS_PER_UNIT);
  const int n_nt = int((P.n_cols + LM_BN - 1) / LM_BN);
  // work unit u = (row block u / n_split, vocabulary split u % n_split)
  const int n_split = P.n_split;
  const int n_units = n_mb * n_split;
  // kSpMajor: units ordered split-major, so the CTAs resident at once share a
  // vocabulary range and each W tile is fetched from DRAM once per wave and
  // served to the other CTAs from L2 (row-block-major otherwise)
  auto unit_tiles = [&](int u, int& mb, int& nt0, int& nt1) {
    int sp;
    if (P.sp_major) {
      sp = u / n_mb;
      mb = u - sp * n_mb;
    } else {
      mb = u / n_split;
      sp = u - mb * n_split;
    }
    nt0 = int((int64_t(sp) * n_nt) / n_split);
    nt1 = int((int64_t(sp + 1) * n_nt) / n_split);
    return sp;
  };
  const int n_kb = int(P.dim / LM_BK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&tail->full[i], 1);
      mbar_init(&tail->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tail->tfull[i], 1);
      mbar_init(&tail->tempty[i], kPair ? 8 : 4);  // epilogue warps of the pair / of the CTA
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tail->tmem_base)),
                   "r"(LM_TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tail->tmem_base)),
                   "r"(LM_TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tail->tmem_base;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (int u = unit0; u < n_units; u += unit_stride) {
        int mb, nt0, nt1;
        unit_tiles(u, mb, nt0, nt1);
        const int xrow = mb * ROWS_PER_UNIT + int(rank) * LM_BM;
        for (int nt = nt0; nt < nt1; ++nt) {
          const int wrow = int(P.col0) + nt * LM_BN + int(rank) * B_ROWS;
          for (int kb = 0; kb < n_kb; ++kb) {
            lm_wait(smem_u32(&tail->empty[stage]), phase ^ 1u);
            const uint32_t fb = smem_u32(&tail->full[stage]);
            const uint32_t a = ring + stage * STAGE;
            if constexpr (kPair) {
              // both CTAs' bytes complete on the leader's full barrier
              if (leader) lm_expect_tx(fb, 2 * STAGE);
              const uint32_t lfb = lm_peer0(fb);
              lm_tma_2d_pair(a, &tmX, kb * LM_BK, xrow, lfb);
              lm_tma_2d_pair(a + LM_A_BYTES, &tmW, kb * LM_BK, wrow, lfb);
            } else {
              lm_expect_tx(fb, STAGE);
              lm_tma_2d(a, &tmX, kb * LM_BK, xrow, fb);
              lm_tma_2d(a + LM_A_BYTES, &tmW, kb * LM_BK, wrow, fb);
            }
            if (++stage == uint32_t(NST)) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer (leader) ============================
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = lm_idesc_t<kPair>();
      uint32_t stage = 0, phase = 0, tile = 0;
      for (int u = unit0; u < n_units; u += unit_stride) {
        int mb, nt0, nt1;
        unit_tiles(u, mb, nt0, nt1);
        for (int nt = nt0; nt < nt1; ++nt, ++tile) {
          const uint32_t acc = tile & 1u, acc_phase = (tile >> 1) & 1u;
          if constexpr (kPair) {
            while (!mbar_try_wait_cluster(smem_u32(&tail->tempty[acc]), acc_phase ^ 1u)) {
            }
          } else {
            lm_wait(smem_u32(&tail->tempty[acc]), acc_phase ^ 1u);
          }
          tc_fence_after();
          const uint32_t d = tmem + acc * LM_BN;
          for (int kb = 0; kb < n_kb; ++kb) {
            lm_wait(smem_u32(&tail->full[stage]), phase);
            tc_fence_after();
            const uint32_t a = ring + stage * STAGE;
            const uint64_t ad = lm_sw128_desc(a), bd = lm_sw128_desc(a + LM_A_BYTES);
#pragma unroll
            for (int k = 0; k < LM_BK / LM_UK; ++k) {  // +32 bytes along K per step
              if constexpr (kPair)
                lm_mma_pair(d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
              else
                lm_mma(d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
            }
            if constexpr (kPair)
              lm_commit_pair(smem_u32(&tail->empty[stage]));
            else
              lm_commit(smem_u32(&tail->empty[stage]));
            if (++stage == uint32_t(NST)) {
              stage = 0;
              phase ^= 1u;
            }
          }
          if constexpr (kPair)
            lm_commit_pair(smem_u32(&tail->tfull[acc]));
          else
            lm_commit(smem_u32(&tail->tfull[acc]));
        }
      }
    }
    __syncwarp();
  } else if (warp >= LM_EPI_WARP0) {
    // ============================ epilogue ============================
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint64_t l2e2 = pk2(kLog2e, kLog2e);
    uint32_t tile = 0;
    if constexpr (kDz) {
      const uint32_t stage_dz = ring + uint32_t(NST * STAGE) + uint32_t(q) * 2u * LM_DZ_TILE_BYTES;
      int sbuf = 0;
      if (lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmD)) : "memory");
      for (int u = unit0; u < n_units; u += unit_stride) {
        int mb, nt0, nt1;
        unit_tiles(u, mb, nt0, nt1);
        const int64_t row = int64_t(mb) * ROWS_PER_UNIT + int64_t(rank) * LM_BM + 32 * q + lane;
        const bool live = row < T;
        const int64_t row0 = row - lane;  // first row of the warp's 32-row slab
        // chunk-relative target column (outside [0, n_cols): no one-hot term here)
        const int64_t yr = live ? int64_t(P.target[row]) - P.col0 : -1;
        const float nl = live ? -P.lse_in[row] * kLog2e : 0.f;
        const float a = live ? P.coef[row] : 0.f, hz = live ? P.coef[T + row] : 0.f;
        const float sy = live ? P.coef[2 * T + row] : 0.f;
        const uint64_t nl2 = pk2(nl, nl), a2 = pk2(a, a), hz2 = pk2(hz, hz);
        for (int nt = nt0; nt < nt1; ++nt, ++tile) {
          const uint32_t acc = tile & 1u, acc_phase = (tile >> 1) & 1u;
          lm_wait_sleep(smem_u32(&tail->tfull[acc]), acc_phase);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < LM_BN; c += 32) {
            float v[32];
            __syncwarp();
            lm_tmem_ld32(tmem + lane_base + acc * LM_BN + uint32_t(c), v);
            const int64_t j0 = int64_t(nt) * LM_BN + c;
            if (j0 >= P.n_cols) continue;  // warp-uniform: the whole tile is past the chunk
            float d[32];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const uint64_t x = pk2(v[i], v[i + 1]);
              const uint64_t p = ex2x2(fma2(x, l2e2, nl2));
              upk2(mul2(p, fma2(hz2, x, a2)), d[i], d[i + 1]);
            }
            if (yr >= j0 && yr < j0 + 32) {
              const int yo = int(yr - j0);
#pragma unroll
              for (int i = 0; i < 32; ++i)
                asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\t@p sub.f32 %0, %0, %3;\n\t}"
                    : "+f"(d[i])
                    : "r"(yo), "r"(i), "f"(sy));
            }
            // stage the warp's [32 rows x 32 columns] bf16 tile (64-byte swizzle:
            // 16-byte granule g of row r at g ^ ((r >> 1) & 3), conflict-free) and
            // let one lane TMA-store it; rows >= T / columns >= n_cols are clipped
            const uint32_t buf = stage_dz + uint32_t(sbuf) * LM_DZ_TILE_BYTES;
            if (lane == 0) lm_store_wait_read<1>();  // this buffer's previous store has read it
            __syncwarp();
            if (live) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t g = uint32_t(k) ^ ((uint32_t(lane) >> 1) & 3u);
                st_shared_v4(buf + uint32_t(lane) * 64u + g * 16u,
                             Vec<bf16_t>::pack2(d[8 * k], d[8 * k + 1]),
                             Vec<bf16_t>::pack2(d[8 * k + 2], d[8 * k + 3]),
                             Vec<bf16_t>::pack2(d[8 * k + 4], d[8 * k + 5]),
                             Vec<bf16_t>::pack2(d[8 * k + 6], d[8 * k + 7]));
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) lm_tma_store_2d(&tmD, buf, int(j0), int(row0));
            sbuf ^= 1;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair)
              lm_arrive_cluster(lm_peer0(smem_u32(&tail->tempty[acc])));
            else
              mbar_arrive(&tail->tempty[acc]);
          }
        }
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    } else
    for (int u = unit0; u < n_units; u += unit_stride) {
      int mb, nt0, nt1;
      const int sp_u = unit_tiles(u, mb, nt0, nt1);
      const int64_t row = int64_t(mb) * ROWS_PER_UNIT + int64_t(rank) * LM_BM + 32 * q + lane;
      const int y = (row < T && P.target) ? P.target[row] : -1;
      float m = -1.0e30f, zy = kNegInf;
      uint64_t s2 = pk2(0.f, 0.f), t2 = pk2(0.f, 0.f);
      for (int nt = nt0; nt < nt1; ++nt, ++tile) {
        const uint32_t acc = tile & 1u, acc_phase = (tile >> 1) & 1u;
        lm_wait_sleep(smem_u32(&tail->tfull[acc]), acc_phase);
        tc_fence_after();
        const int col_tile = nt * LM_BN;
        // two-level sums (32-column chunk, then tile) keep the fp32 rounding of
        // the ~V/2 terms per lane near (32 + 8 + V/256) ulp instead of V/2 ulp
        uint64_t ts2 = pk2(0.f, 0.f), tt2 = pk2(0.f, 0.f);
#pragma unroll 1
        for (int c = 0; c < LM_BN; c += 32) {
          float v[32];
          lm_tmem_ld32(tmem + lane_base + acc * LM_BN + uint32_t(c), v);
          const int col0 = col_tile + c;
          if (col0 + 32 > V) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i >= V) v[i] = -1.0e30f;
          }
          if (y >= col0 && y < col0 + 32) {
            // predicated selects (an indexed read would push v[] to local memory)
            const int yo = y - col0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\tselp.f32 %0, %3, %0, p;\n\t}"
                  : "+f"(zy)
                  : "r"(yo), "r"(i), "f"(v[i]));
          }
          float cm = v[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) cm = fmaxf(cm, v[i]);
          if (cm > m) {  // exact running max (rescale the sums)
            const float sc = ex2((m - cm) * kLog2e);
            const uint64_t sc2 = pk2(sc, sc);
            s2 = mul2(s2, sc2);
            t2 = mul2(t2, sc2);
            ts2 = mul2(ts2, sc2);
            tt2 = mul2(tt2, sc2);
            m = cm;
          }
          const float nmL = -m * kLog2e;
          const uint64_t nm2 = pk2(nmL, nmL);
          uint64_t cs2, ct2;
          {
            const uint64_t x = pk2(v[0], v[1]);
            cs2 = ex2x2(fma2(x, l2e2, nm2));
            ct2 = mul2(cs2, x);
          }
#pragma unroll
          for (int i = 2; i < 32; i += 2) {
            const uint64_t x = pk2(v[i], v[i + 1]);
            const uint64_t p = ex2x2(fma2(x, l2e2, nm2));
            cs2 = add2(cs2, p);
            ct2 = fma2(p, x, ct2);
          }
          ts2 = add2(ts2, cs2);
          tt2 = add2(tt2, ct2);
        }
        s2 = add2(s2, ts2);
        t2 = add2(t2, tt2);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair)
            lm_arrive_cluster(lm_peer0(smem_u32(&tail->tempty[acc])));
          else
            mbar_arrive(&tail->tempty[acc]);
        }
      }
      if (row < T) {
        float s0, s1, t0, t1;
        upk2(s2, s0, s1);
        upk2(t2, t0, t1);
        const float s = s0 + s1, t = t0 + t1;
        if (n_split > 1) {
          P.partial[int64_t(sp_u) * T + row] = make_float4(m, s, t, zy);
        } else {
          const float l = m + logf(s);
          P.lse[row] = l;
          P.ent[row] = l - t / s;
          if (P.lp) P.lp[row] = (y >= 0 && y < V) ? zy - l : kNegInf;
        }
      }
    }
  }
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync_all();  // the peer's MMAs and remote arrivals are done
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(LM_TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(LM_TMEM_COLS)
                   : "memory");
  }
}

// fixed-order merge of the vocabulary-split partials of each row
__global__ void k_lmhead_merge(const LmParams P) {
  const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= P.n_rows) return;
  Online o = {kNegInf, 0.f, 0.f};
  float zy = kNegInf;
  for (int sp = 0; sp < P.n_split; ++sp) {
    const float4 w = P.partial[int64_t(sp) * P.n_rows + row];
    o = online_merge(o, Online{w.x, w.y, w.z});
    zy = fmaxf(zy, w.w);
  }
  const float l = o.m + logf(o.s);
  P.lse[row] = l;
  P.ent[row] = l - o.t / o.s;
  if (P.lp) {
    const int y = P.target[row];
    P.lp[row] = (y >= 0 && y < P.vocab) ? zy - l : kNegInf;
  }
}

// 2-CTA pairs by default, forward and backward (dz) chunks: each SM stages and
// reads half of the W tile, and ncu shows the single-CTA forward with its
// tensor-memory operand path 92-94 % busy (profiles/r02_lmhead_fwd_ab.txt).
// Round-2 A/B, 16,384 rows (same box): forward 1,620 vs 1,558 TFLOP/s at
// d = 1536 (split-major), 1,412 vs 1,376 at d = 3584 (row-block-major); round 1
// measured the dz chunks +9 % (profiles/r01_lmhead_bwd.txt).  TG_LMHEAD_PAIR=0/1
// forces one mode for both (A/B build).
static bool lm_pair_mode(bool dz = false) {
  (void)dz;
  static int mode = -2;
  if (mode == -2) {
    const int v = ab_env("TG_LMHEAD_PAIR", -1);  // A/B build only
    mode = v < 0 ? -1 : (v != 0);
  }
  return mode != 0;
}

// Work-unit order.  Split-major when the CTAs resident at once (one 128-row X
// block each, all on the same vocabulary range) keep their X blocks and the
// W range in L2 -- each W tile then comes from DRAM once and is served to the
// other CTAs from L2; row-block-major otherwise (a few X blocks, the CTAs that
// share a range walk the W tiles in step).  Measured (profiles/r01_lmhead_bwd.txt):
// split-major +3 % at d = 1,536 (116 MB working set), -20 % at d = 3,584
// (272 MB).  TG_LMHEAD_ORDER=0/1 forces one order.
static int lm_sp_major(int64_t cols, int64_t dim, int n_split, int n_sms) {
  static int mode = -2;
  if (mode == -2) {
    const int v = ab_env("TG_LMHEAD_ORDER", -1);  // A/B build only
    mode = v < 0 ? -1 : (v != 0);
  }
  if (mode >= 0) return mode;
  const double ws = 2.0 * double(dim) * (double(n_sms) * LM_BM + double(cols) / n_split);
  return ws <= 120.0 * 1024 * 1024 ? 1 : 0;
}

// Vocabulary splits per row block: enough work units to fill the SMs (or SM
// pairs) in whole waves -- small row counts would otherwise leave SMs idle.
int lm_split(int64_t n_rows, int64_t vocab, int n_sms, bool pair) {
  const int64_t rows_per_unit = pair ? 2 * LM_BM : LM_BM;
  const int64_t slots = pair ? n_sms / 2 : n_sms;
  const int64_t n_mb = (n_rows + rows_per_unit - 1) / rows_per_unit;
  const int64_t n_nt = (vocab + LM_BN - 1) / LM_BN;
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= 16 && sp <= n_nt; ++sp) {
    const int64_t units = n_mb * sp;
    const int64_t waves = (units + slots - 1) / slots;
    const double eff = double(units) / double(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = sp;
    }
  }
  return best;
}

int lm_split(int64_t n_rows, int64_t vocab, int n_sms) {
  return lm_split(n_rows, vocab, n_sms, lm_pair_mode());
}

size_t lm_workspace_bytes(int64_t n_rows, int64_t vocab, int n_sms) {
  const int sp = lm_split(n_rows, vocab, n_sms);
  return sp > 1 ? size_t(sp) * size_t(n_rows) * sizeof(float4) : 0;
}

// ---- host side --------------------------------------------------------------------

template <bool kDz>
static cudaError_t lm_launch(const CUtensorMap& mx, const CUtensorMap& mw, const CUtensorMap& md,
                             const LmParams& P, bool pair, int n_sms, cudaStream_t stream) {
  cudaError_t e;
  if (pair) {
    const size_t smem = lm_smem_bytes<true>();
    e = cudaFuncSetAttribute(k_lmhead_logprob<true, kDz>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const int64_t units = ((P.n_rows + 2 * LM_BM - 1) / (2 * LM_BM)) * P.n_split;
    const int64_t pairs = units < n_sms / 2 ? units : n_sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * pairs));
    cfg.blockDim = dim3(LM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_lmhead_logprob<true, kDz>, mx, mw, md, P);
  }
  const size_t smem = lm_smem_bytes<false>();
  e = cudaFuncSetAttribute(k_lmhead_logprob<false, kDz>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int64_t units = ((P.n_rows + LM_BM - 1) / LM_BM) * P.n_split;
  const int grid = int(units < n_sms ? units : n_sms);
  k_lmhead_logprob<false, kDz><<<grid, LM_THREADS, smem, stream>>>(mx, mw, md, P);
  return cudaGetLastError();
}

// returns a cudaError_t; cudaErrorNotSupported when the driver entry point is missing
cudaError_t launch_lmhead_logprob(const void* hidden, int64_t ld_hidden, const void* weight,
                                  int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                                  const int32_t* target, float* lp, float* ent, float* lse,
                                  void* workspace, size_t workspace_bytes, int n_sms,
                                  cudaStream_t stream) {
  const bool pair = lm_pair_mode();
  CUtensorMap mx, mw;
  if (!lm_make_map(&mx, hidden, n_rows, dim, ld_hidden, LM_BM)) return cudaErrorNotSupported;
  if (!lm_make_map(&mw, weight, vocab, dim, ld_weight, pair ? LM_BN / 2 : LM_BN))
    return cudaErrorNotSupported;
  LmParams P = {};
  P.n_rows = n_rows;
  P.vocab = vocab;
  P.dim = dim;
  P.col0 = 0;
  P.n_cols = vocab;
  P.target = target;
  P.lp = lp;
  P.ent = ent;
  P.lse = lse;
  P.n_split = lm_split(n_rows, vocab, n_sms);
  P.sp_major = lm_sp_major(vocab, dim, P.n_split, n_sms);
  P.partial = reinterpret_cast<float4*>(workspace);
  if (P.n_split > 1 && (!workspace || workspace_bytes < lm_workspace_bytes(n_rows, vocab, n_sms)))
    return cudaErrorInvalidValue;
  cudaError_t e = lm_launch<false>(mx, mw, mx, P, pair, n_sms, stream);  // no dz map
  if (e != cudaSuccess) return e;
  if (P.n_split > 1) k_lmhead_merge<<<int((n_rows + 255) / 256), 256, 0, stream>>>(P);
  return cudaGetLastError();
}

// backward of one vocabulary chunk [col0, col0 + n_cols): bf16 dz tiles, no
// workspace (tiles are independent; the split only fills the SMs)
cudaError_t launch_lmhead_dz(const void* hidden, int64_t ld_hidden, const void* weight,
                             int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                             int64_t col0, int64_t n_cols, const int32_t* target,
                             const float* lse, const float* coef, void* dz, int64_t ld_dz,
                             int n_sms, cudaStream_t stream) {
  const bool pair = lm_pair_mode(true);
  CUtensorMap mx, mw;
  if (!lm_make_map(&mx, hidden, n_rows, dim, ld_hidden, LM_BM)) return cudaErrorNotSupported;
  if (!lm_make_map(&mw, weight, vocab, dim, ld_weight, pair ? LM_BN / 2 : LM_BN))
    return cudaErrorNotSupported;
  LmParams P = {};
  P.n_rows = n_rows;
  P.vocab = vocab;
  P.dim = dim;
  P.col0 = col0;
  P.n_cols = n_cols;
  P.target = target;
  P.lse_in = lse;
  P.coef = coef;
  P.dz = reinterpret_cast<uint16_t*>(dz);
  P.ld_dz = ld_dz;
  P.n_split = lm_split(n_rows, n_cols, n_sms, pair);
  P.sp_major = lm_sp_major(n_cols, dim, P.n_split, n_sms);
  CUtensorMap md;
  if (!lm_make_map(&md, dz, n_rows, n_cols, ld_dz, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorNotSupported;
  return lm_launch<true>(mx, mw, md, P, pair, n_sms, stream);
}

}  // namespace tg
