// tg_gemm.cu -- K8: the LM-head backward GEMMs on the 5th-gen tensor cores.
//
// SURVEY.md §8(f-1), consumer side: with the vocabulary-chunked backward
// (tg_lmhead_dlogits writes dz = d loss / d z of one chunk [T, n] in bf16) the
// gradients w.r.t. the LM-head inputs are two GEMMs per chunk
//     d hidden [T, d] (+)= dz [T, n] . W_c [n, d]         A K-major,  B MN-major
//     d W_c    [n, d]   = dz^T [n, T] . hidden [T, d]     A MN-major, B MN-major
// (the analogue of SparseGrad.add_row + apply_update behind an LM head,
// policy.py:215-250 / algorithms.py:329-348).  Both run here on tcgen05 with
// TMA-fed shared-memory rings -- no cuBLAS on the path.
//
// Design (sm_100a, one persistent CTA per SM, 128 x 256 output tiles):
//  * warp 0 / one lane: TMA producer.  A K-major operand tile is one box
//    [128 rows x 64 K] (128-byte swizzle); an MN-major one is [64 K rows x 64
//    MN] boxes side by side (2 for A, 4 for B), each 8 KB: the UMMA descriptor's
//    LBO steps between them, SBO (1 KB) between 8-row K groups.  4 stages of
//    48 KB, full / empty mbarriers.
//  * warp 1 / one lane: tcgen05.mma.cta_group::1.kind::f16 (M 128, N 256,
//    K 16) into one of two TMEM accumulators (2 x 256 fp32 columns), with
//    tcgen05.commit releasing ring slots and publishing finished tiles.
//  * warp 2: TMEM allocation.  Warps 4..7: epilogue -- tcgen05.ld of the
//    warp's 32-lane quadrant (row = lane), then fp32 read-modify-write (d hidden
//    accumulates over the vocabulary chunks) or bf16 stores (d W), whole
//    128-byte lines per thread; the other accumulator takes the next tile's MMAs.
//  * tile order n-fastest: the CTAs resident at once share A strips (and the
//    B operand of one chunk fits L2), so DRAM sees each operand about once.
//  * both GEMMs of a chunk can share one launch (tg_lmhead_grad_chunk): one
//    tile queue, so neither GEMM's last partial wave idles the SMs.
#include "tg_common.cuh"
#include "tg_umma.cuh"
#include "tg_vecmath.cuh"

namespace tg {

constexpr int G_BM = 128;
constexpr int G_BN = 256;
constexpr int G_BK = 64;
constexpr int G_UK = 16;
constexpr int G_A_BYTES = G_BM * G_BK * 2;  // 16 KB
constexpr int G_THREADS = 256;
constexpr int G_BOX = 64 * 64 * 2;          // one MN-major box [64 K][64 MN]: 8 KB
#ifndef TG_GEMM_PAIR_STAGES
#define TG_GEMM_PAIR_STAGES 6
#endif
constexpr int G_MAX_STAGES = TG_GEMM_PAIR_STAGES > 4 ? TG_GEMM_PAIR_STAGES : 4;
// kPair = false: one CTA per 128 x 256 tile (cta_group::1), 4 stages of 48 KB.
// kPair = true : a 2-CTA cluster per 256 x 256 tile (cta_group::2, M 256): each
//   CTA stages its own 128 A rows and half of the B tile (128 N), so a stage is
//   32 KB and 6 fit -- per SM the B bytes staged and read halve.
template <bool kPair> constexpr int g_b_rows() { return kPair ? G_BN / 2 : G_BN; }
template <bool kPair> constexpr int g_stage() { return G_A_BYTES + g_b_rows<kPair>() * G_BK * 2; }
template <bool kPair> constexpr int g_stages() { return kPair ? TG_GEMM_PAIR_STAGES : 4; }
template <bool kPair> constexpr int g_tile_m() { return kPair ? 2 * G_BM : G_BM; }

// One GEMM of a launch: D [M, N] (+)= A . B, operand majors, output type.
struct GemmJob {
  int64_t M, N, K;
  void* out;          // fp32 or bf16 [M, ld_out]
  int64_t ld_out;
  int accumulate;     // fp32 output: D += A.B (else D = A.B)
  int a_mn, b_mn;     // operand majors (0 K-major, 1 MN-major)
  int bf16_out;
};

// Up to two independent GEMMs in one persistent launch (d hidden and d W of a
// vocabulary chunk): their tiles form one queue, so the tail of one fills the
// SMs with tiles of the other (2 x 768 tiles at T = 16 k, d = 1,536 are 10.4
// waves of 148 instead of 5.2, 94 % instead of 86 % of the last wave busy).
struct GemmParams {
  GemmJob job[2];
  int n_jobs;
  // Tail split: the last n_half tiles of the queue (those of the final,
  // partial wave, when they fill at most half of it) run as two 256 x 128
  // half tiles each -- the last wave then takes half as long.  Work item w <
  // n_tiles - n_half is tile w; the 2 n_half items after it are the halves.
  int n_half;
};

struct GemmSmemTail {
  uint64_t full[G_MAX_STAGES];
  uint64_t empty[G_MAX_STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

template <bool kPair>
size_t gemm_smem_bytes() {
  return size_t(g_stages<kPair>()) * g_stage<kPair>() + sizeof(GemmSmemTail) + 1024;
}

// tile t of the queue -> (job, m0, n0, width)
struct TileRef {
  int j;
  int64_t m0, n0;
  int nw;  // N columns of the tile (G_BN, or G_BN / 2 for a tail half)
};

// (m0: the tile's first row; a pair's CTA rank r owns rows m0 + 128 r ..)
template <int BM>
__host__ __device__ __forceinline__ TileRef tile_of(const GemmParams& P, int t) {
  const GemmJob& J0 = P.job[0];
  const int nn0 = int((J0.N + G_BN - 1) / G_BN);
  const int t0 = int((J0.M + BM - 1) / BM) * nn0;
  TileRef r;
  if (t < t0) {
    r.j = 0;
    r.m0 = int64_t(t / nn0) * BM;
    r.n0 = int64_t(t % nn0) * G_BN;
  } else {
    const int u = t - t0;
    const int nn1 = int((P.job[1].N + G_BN - 1) / G_BN);
    r.j = 1;
    r.m0 = int64_t(u / nn1) * BM;
    r.n0 = int64_t(u % nn1) * G_BN;
  }
  r.nw = G_BN;
  return r;
}

// work item w of a launch with n_tiles tiles and the last P.n_half split
template <int BM>
__host__ __device__ __forceinline__ TileRef item_of(const GemmParams& P, int n_tiles, int w) {
  const int first_half = n_tiles - P.n_half;
  if (w < first_half) return tile_of<BM>(P, w);
  const int h = w - first_half;
  TileRef r = tile_of<BM>(P, first_half + h / 2);
  r.n0 += int64_t(h & 1) * (G_BN / 2);
  r.nw = G_BN / 2;
  return r;
}

template <int BM>
__host__ __device__ __forceinline__ int n_tiles_of(const GemmJob& J) {
  return int(((J.M + BM - 1) / BM) * ((J.N + G_BN - 1) / G_BN));
}

template <bool kPair>
__global__ void __launch_bounds__(G_THREADS, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                const GemmParams P) {
  constexpr int STAGE = g_stage<kPair>();
  constexpr int NST = g_stages<kPair>();
  constexpr int BM = g_tile_m<kPair>();       // output rows per tile (both CTAs of a pair)
  constexpr int B_ROWS = g_b_rows<kPair>();   // B (N) columns staged per CTA
  extern __shared__ __align__(1024) unsigned char g_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(g_smem_raw) + 1023) & ~uintptr_t(1023));
  GemmSmemTail* tail = reinterpret_cast<GemmSmemTail*>(smem + size_t(NST) * STAGE);
  const uint32_t ring = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int tile0 = kPair ? int(cluster_id_x()) : int(blockIdx.x);
  const int tile_stride = kPair ? int(n_clusters_x()) : int(gridDim.x);
  const int n_tiles = n_tiles_of<BM>(P.job[0]) + (P.n_jobs > 1 ? n_tiles_of<BM>(P.job[1]) : 0);
  const int n_items = n_tiles + P.n_half;

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
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&tail->tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&tail->tmem_base))
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
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
      if (P.n_jobs > 1) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA1)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB1)) : "memory");
      }
      uint32_t stage = 0, phase = 0;
      for (int t = tile0; t < n_items; t += tile_stride) {
        const TileRef tr = item_of<BM>(P, n_tiles, t);
        const GemmJob J = tr.j ? P.job[1] : P.job[0];
        const CUtensorMap* mA = tr.j ? &tmA1 : &tmA0;
        const CUtensorMap* mB = tr.j ? &tmB1 : &tmB0;
        // this CTA's A rows and B columns of the tile (a tail half: half of them)
        const int b_rows = tr.nw == G_BN ? B_ROWS : B_ROWS / 2;
        const int m0 = int(tr.m0) + int(rank) * G_BM, n0 = int(tr.n0) + int(rank) * b_rows;
        const uint32_t stage_bytes = uint32_t(G_A_BYTES + b_rows * G_BK * 2);
        const int n_kb = int((J.K + G_BK - 1) / G_BK);
        for (int kb = 0; kb < n_kb; ++kb) {
          lm_wait(smem_u32(&tail->empty[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&tail->full[stage]);
          const uint32_t a = ring + stage * STAGE, b = a + G_A_BYTES;
          const int k0 = kb * G_BK;
          // pair: both CTAs' bytes complete on the leader's full barrier
          uint32_t bar = fb;
          if constexpr (kPair) {
            if (leader) lm_expect_tx(fb, 2 * stage_bytes);
            bar = lm_peer0(fb);
          } else {
            lm_expect_tx(fb, stage_bytes);
          }
          auto load = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
            if constexpr (kPair)
              lm_tma_2d_pair(dst, m, c0, c1, bar);
            else
              lm_tma_2d(dst, m, c0, c1, bar);
          };
          if (J.a_mn) {
#pragma unroll
            for (int j = 0; j < G_BM / 64; ++j) load(a + j * G_BOX, mA, m0 + 64 * j, k0);
          } else {
            load(a, mA, k0, m0);
          }
          if (J.b_mn) {
#pragma unroll
            for (int j = 0; j < B_ROWS / 64; ++j)
              if (64 * j < b_rows) load(b + j * G_BOX, mB, n0 + 64 * j, k0);
          } else {
            load(b, mB, k0, n0);
          }
          if (++stage == uint32_t(NST)) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer (pair: the leader) ============================
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, tile = 0;
      for (int t = tile0; t < n_items; t += tile_stride, ++tile) {
        const TileRef tr = item_of<BM>(P, n_tiles, t);
        const GemmJob J = tr.j ? P.job[1] : P.job[0];
        const bool amn = J.a_mn != 0, bmn = J.b_mn != 0;
        const uint32_t idesc = umma_idesc_bf16(BM, tr.nw, amn, bmn);
        // descriptor address step per K = 16: 32 B (K-major) or 16 rows x 128 B (MN-major)
        const uint64_t a_step = amn ? 128u : 2u, b_step = bmn ? 128u : 2u;
        const int n_kb = int((J.K + G_BK - 1) / G_BK);
        const uint32_t acc = tile & 1u, acc_phase = (tile >> 1) & 1u;
        if constexpr (kPair) {
          while (!mbar_try_wait_cluster(smem_u32(&tail->tempty[acc]), acc_phase ^ 1u)) {
          }
        } else {
          lm_wait(smem_u32(&tail->tempty[acc]), acc_phase ^ 1u);
        }
        tc_fence_after();
        const uint32_t d = tmem + acc * G_BN;
        for (int kb = 0; kb < n_kb; ++kb) {
          lm_wait(smem_u32(&tail->full[stage]), phase);
          tc_fence_after();
          const uint32_t a = ring + stage * STAGE, b = a + G_A_BYTES;
          const uint64_t ad = amn ? lm_sw128_mn_desc(a, G_BOX) : lm_sw128_desc(a);
          const uint64_t bd = bmn ? lm_sw128_mn_desc(b, G_BOX) : lm_sw128_desc(b);
#pragma unroll
          for (int k = 0; k < G_BK / G_UK; ++k) {
            if constexpr (kPair)
              lm_mma_pair(d, ad + a_step * k, bd + b_step * k, idesc, (kb | k) != 0);
            else
              lm_mma(d, ad + a_step * k, bd + b_step * k, idesc, (kb | k) != 0);
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
    __syncwarp();
  } else if (warp >= 4) {
    // ============================ epilogue ============================
    const int q = warp & 3;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    uint32_t tile = 0;
    for (int t = tile0; t < n_items; t += tile_stride, ++tile) {
      const TileRef tr = item_of<BM>(P, n_tiles, t);
      const GemmJob J = tr.j ? P.job[1] : P.job[0];
      const uint32_t acc = tile & 1u, acc_phase = (tile >> 1) & 1u;
      const int64_t row = tr.m0 + int64_t(rank) * G_BM + 32 * q + lane;
      lm_wait_sleep(smem_u32(&tail->tfull[acc]), acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < tr.nw; c += 32) {
        float v[32];
        __syncwarp();
        lm_tmem_ld32(tmem + lane_base + acc * G_BN + uint32_t(c), v);
        const int64_t col = tr.n0 + c;
        if (row >= J.M || col >= J.N) continue;  // N is a multiple of 32 (host check)
        if (J.bf16_out) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(J.out) +
                                                row * J.ld_out + col);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            dst[k] = make_uint4(Vec<bf16_t>::pack2(v[8 * k], v[8 * k + 1]),
                                Vec<bf16_t>::pack2(v[8 * k + 2], v[8 * k + 3]),
                                Vec<bf16_t>::pack2(v[8 * k + 4], v[8 * k + 5]),
                                Vec<bf16_t>::pack2(v[8 * k + 6], v[8 * k + 7]));
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(J.out) +
                                                  row * J.ld_out + col);
          if (J.accumulate) {
            float4 o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = dst[k];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              dst[k] = make_float4(o[k].x + v[4 * k], o[k].y + v[4 * k + 1], o[k].z + v[4 * k + 2],
                                   o[k].w + v[4 * k + 3]);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              dst[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          }
        }
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
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync_all();  // no CTA frees its TMEM / leaves while the pair still uses it
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// tail split on by default (TG_GEMM_TAIL=0 turns it off, A/B build)
static bool gemm_tail_split() {
  static int mode = -2;
  if (mode == -2) mode = ab_env("TG_GEMM_TAIL", 1);
  return mode != 0;
}

// 2-CTA pairs by default (TG_GEMM_PAIR=0 forces single CTAs, A/B build)
static bool gemm_pair_mode() {
  static int mode = -2;
  if (mode == -2) mode = ab_env("TG_GEMM_PAIR", 1);
  return mode != 0;
}

template <bool kPair>
static cudaError_t gemm_launch_t(const CUtensorMap (&maps)[4], const GemmParams& P, int n_sms,
                                 cudaStream_t stream) {
  const size_t smem = gemm_smem_bytes<kPair>();
  cudaError_t e = cudaFuncSetAttribute(k_gemm_bf16<kPair>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  constexpr int BM = g_tile_m<kPair>();
  int64_t tiles = 0;
  bool b_mn_all = true;  // the half tiles load MN-major B boxes (64 columns each)
  for (int j = 0; j < P.n_jobs; ++j) {
    tiles += n_tiles_of<BM>(P.job[j]);
    b_mn_all &= P.job[j].b_mn != 0;
  }
  const int64_t slots = kPair ? n_sms / 2 : n_sms;
  // tail split: a last wave at most half full runs as half tiles
  GemmParams Q = P;
  const int64_t rem = tiles % slots;
  Q.n_half = (gemm_tail_split() && b_mn_all && rem > 0 && 2 * rem <= slots) ? int(rem) : 0;
  const int64_t items = tiles + Q.n_half;
  const int units = int(items < slots ? items : slots);
  if (units <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(kPair ? 2 * units : units));
  cfg.blockDim = dim3(G_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_bf16<kPair>, maps[0], maps[1], maps[2], maps[3], Q);
}

static cudaError_t gemm_launch(const CUtensorMap (&maps)[4], const GemmParams& P, int n_sms,
                               cudaStream_t stream) {
  return gemm_pair_mode() ? gemm_launch_t<true>(maps, P, n_sms, stream)
                          : gemm_launch_t<false>(maps, P, n_sms, stream);
}

// d hidden [T, d] (+)= dz [T, n] . W[col0 : col0 + n]: A dz K-major (box [128
// rows][64 K]), B the chunk's W rows MN-major (boxes [64 K][64 N]); fp32 out
static bool job_grad_hidden(GemmJob& J, CUtensorMap& ma, CUtensorMap& mb, const void* dz,
                            int64_t ld_dz, const void* weight, int64_t ld_weight, int64_t n_rows,
                            int64_t n_cols, int64_t dim, int64_t col0, float* d_hidden,
                            int64_t ld_dh, int accumulate) {
  if (!lm_make_map(&ma, dz, n_rows, n_cols, ld_dz, G_BM)) return false;
  const void* wc = reinterpret_cast<const uint16_t*>(weight) + col0 * ld_weight;
  if (!lm_make_map(&mb, wc, n_cols, dim, ld_weight, 64)) return false;
  J = GemmJob{n_rows, dim, n_cols, d_hidden, ld_dh, accumulate, 0, 1, 0};
  return true;
}

// d W[col0 : col0 + n] [n, d] = dz^T [n, T] . hidden [T, d]: A dz^T MN-major
// (boxes [64 K = dz rows][64 M = dz columns]), B hidden MN-major; bf16 out
static bool job_grad_weight(GemmJob& J, CUtensorMap& ma, CUtensorMap& mb, const void* dz,
                            int64_t ld_dz, const void* hidden, int64_t ld_hidden, int64_t n_rows,
                            int64_t n_cols, int64_t dim, void* d_weight, int64_t ld_dw) {
  if (!lm_make_map(&ma, dz, n_rows, n_cols, ld_dz, 64)) return false;
  if (!lm_make_map(&mb, hidden, n_rows, dim, ld_hidden, 64)) return false;
  J = GemmJob{n_cols, dim, n_rows, d_weight, ld_dw, 0, 1, 1, 1};
  return true;
}

cudaError_t launch_grad_hidden(const void* dz, int64_t ld_dz, const void* weight,
                               int64_t ld_weight, int64_t n_rows, int64_t n_cols, int64_t dim,
                               int64_t col0, float* d_hidden, int64_t ld_dh, int accumulate,
                               int n_sms, cudaStream_t stream) {
  CUtensorMap maps[4];
  GemmParams P = {};
  if (!job_grad_hidden(P.job[0], maps[0], maps[1], dz, ld_dz, weight, ld_weight, n_rows, n_cols,
                       dim, col0, d_hidden, ld_dh, accumulate))
    return cudaErrorNotSupported;
  maps[2] = maps[0];
  maps[3] = maps[1];
  P.n_jobs = 1;
  return gemm_launch(maps, P, n_sms, stream);
}

cudaError_t launch_grad_weight(const void* dz, int64_t ld_dz, const void* hidden,
                               int64_t ld_hidden, int64_t n_rows, int64_t n_cols, int64_t dim,
                               void* d_weight, int64_t ld_dw, int n_sms, cudaStream_t stream) {
  CUtensorMap maps[4];
  GemmParams P = {};
  if (!job_grad_weight(P.job[0], maps[0], maps[1], dz, ld_dz, hidden, ld_hidden, n_rows, n_cols,
                       dim, d_weight, ld_dw))
    return cudaErrorNotSupported;
  maps[2] = maps[0];
  maps[3] = maps[1];
  P.n_jobs = 1;
  return gemm_launch(maps, P, n_sms, stream);
}

// both GEMMs of one chunk in one launch (the job with the longer K first)
cudaError_t launch_grad_chunk(const void* dz, int64_t ld_dz, const void* hidden,
                              int64_t ld_hidden, const void* weight, int64_t ld_weight,
                              int64_t n_rows, int64_t n_cols, int64_t dim, int64_t col0,
                              float* d_hidden, int64_t ld_dh, int accumulate, void* d_weight,
                              int64_t ld_dw, int n_sms, cudaStream_t stream) {
  CUtensorMap maps[4];
  GemmParams P = {};
  const int ih = n_cols >= n_rows ? 0 : 1;  // d hidden's K = n_cols, d W's K = n_rows
  if (!job_grad_hidden(P.job[ih], maps[2 * ih], maps[2 * ih + 1], dz, ld_dz, weight, ld_weight,
                       n_rows, n_cols, dim, col0, d_hidden, ld_dh, accumulate) ||
      !job_grad_weight(P.job[1 - ih], maps[2 - 2 * ih], maps[3 - 2 * ih], dz, ld_dz, hidden,
                       ld_hidden, n_rows, n_cols, dim, d_weight, ld_dw))
    return cudaErrorNotSupported;
  P.n_jobs = 2;
  return gemm_launch(maps, P, n_sms, stream);
}

}  // namespace tg
