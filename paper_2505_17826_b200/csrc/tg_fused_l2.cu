// tg_fused_l2.cu -- K1 alternative: fused single-pass loss with the row's
// second read served by L2 instead of shared memory (A/B against
// tg_fused_tma.cu; selected with TG_FUSED_IMPL=l2).
//
// One persistent 1024-thread CTA per SM owns whole rows.  Phase 1 streams the
// row from HBM with 128-bit loads tagged L2::evict_last (four in flight per
// thread) and reduces (max, sum e, sum e z); phase 2 re-reads the row -- an L2
// hit, since the chip-wide live set is one row per SM (~44 MB at V = 151,936,
// well inside the 126 MB L2) -- with L2::evict_first and writes dz with
// streaming stores.  HBM traffic stays 4V bytes per row when the re-read
// hits; there is no cluster exchange, no ring and no per-chunk barrier.
#include <stdlib.h>

#include "tg_common.cuh"
#include "tg_rowcoef.cuh"
#include "tg_vecmath.cuh"

namespace tg {

constexpr int kL2Vec = 4;  // vectors per thread per iteration

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint4 ld_hint(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

template <typename T, int kL2Threads>
__global__ void __launch_bounds__(kL2Threads, 1024 / kL2Threads)
    k_fused_l2(const KParams P, const RowMeta* __restrict__ meta, int prefetch) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  constexpr int kL2Warps = kL2Threads / 32;
  __shared__ float4 red[kL2Warps];
  __shared__ float4 bc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int V = int(P.vocab);
  const int nvec = (V + EPV - 1) / EPV;
  const int tail_vec = (V % EPV) ? nvec - 1 : -1;
  const int tail_valid = V - (nvec - 1) * EPV;
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  __shared__ double sd[15];  // per-CTA stats, touched by thread 0 only
  if (tid < 15) sd[tid] = 0.0;
  auto row_ptr = [&](int64_t row) {
    const int64_t src = P.row_index ? P.row_index[row] : row;
    return reinterpret_cast<const char*>(P.logits) + src * P.ld * ESZ;
  };
  for (int64_t row = blockIdx.x; row < P.n_rows; row += gridDim.x) {
    const char* zrow = row_ptr(row);
    RowMeta cur;
    if (tid == 0) cur = load_meta(meta, row);
    // ---------------- phase 1 (HBM -> registers, lines kept in L2) -------------
    Acc2 acc = {kNegInf, pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f)};
    for (int base = 0; base < nvec; base += kL2Threads * kL2Vec) {
      uint4 u[kL2Vec];
      bool valid[kL2Vec];
#pragma unroll
      for (int g = 0; g < kL2Vec; ++g) {
        const int vec = base + g * kL2Threads + tid;
        valid[g] = vec < nvec;
        u[g] = valid[g] ? ld_hint(zrow + int64_t(vec) * 16, keep) : Pk<T>::neutral();
      }
#pragma unroll
      for (int g = 0; g < kL2Vec; ++g) {
        Pk<T>::clamp(u[g]);
        if (base + g * kL2Threads + tid == tail_vec) Pk<T>::mask_from(u[g], tail_valid);
      }
      const float vmax = group_max<T>(u);
      if (__any_sync(0xffffffffu, vmax > acc.m + kSlack)) rescale(acc, vmax);
#pragma unroll
      for (int g = 0; g < kL2Vec; ++g)
        if (valid[g]) accumulate<T>(acc, u[g]);
    }
    if (prefetch && tid == 0 && row + gridDim.x < P.n_rows) {
      const char* nz = row_ptr(row + gridDim.x);
      const uint32_t bytes = uint32_t(nvec) * 16u;
      for (uint32_t off = 0; off < bytes; off += 65536u) {
        const uint32_t n = min(65536u, bytes - off);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nz + off), "r"(n)
                     : "memory");
      }
    }
    Online o;
    {
      float s0, s1, t0, t1;
      upk2(acc.s2, s0, s1);
      upk2(acc.t2, t0, t1);
      o = warp_merge(Online{acc.m, s0 + s1, t0 + t1});
    }
    if (lane == 0) red[warp] = make_float4(o.m, o.s, o.t, 0.f);
    __syncthreads();
    if (warp == 0) {
      const float4 v = lane < kL2Warps ? red[lane] : make_float4(kNegInf, 0.f, 0.f, 0.f);
      const Online tot = warp_merge(Online{v.x, v.y, v.z});
      if (lane == 0) {
        const int y = cur.y;
        const bool bad_target = (cur.flags & 2u) != 0;
        const float zy = (!bad_target) ? Vec<T>::load1(zrow, y) : kNegInf;
        const float lse = tot.m + logf(tot.s);
        const float H = lse - tot.t / tot.s;
        const float lp = zy - lse;
        RowTerms t = meta_terms(P, cur, lp, H);
        if (bad_target) {
          t.s = 0.f;
          t.h = 0.f;
        }
        bc = make_float4(t.s + t.h * (H - lse), t.h, lse, t.s);
        P.lp[row] = lp;
        P.ent[row] = H;
        P.lse[row] = lse;
        const bool nonfin = !(finite_f(lse) && finite_f(lp) && finite_f(H) && finite_f(t.s) &&
                              finite_f(t.h));
        sd[0] += t.l_pg;
        sd[1] += t.l_kl;
        sd[2] += t.l_ent;
        sd[3] += t.l_sft;
        sd[4] += t.clipped;
        sd[5] += t.dual;
        if (t.rl) {
          sd[6] += H;
          sd[7] += t.kl;
          sd[8] += t.ppo_kl;
          sd[11] += t.ratio;
          sd[12] += 1.0;
        }
        sd[9] += lp;
        sd[10] += nonfin;
        sd[13] += bad_target;
        sd[14] += 1.0;
      }
    }
    __syncthreads();
    // ---------------- phase 2 (L2 -> dz) ----------------
    const float4 b = bc;
    const float a = b.x, hz = b.y, s_t = b.w, lseL = b.z * kLog2e;
    const uint64_t nl2 = pk2(-lseL, -lseL), av2 = pk2(a, a), hz2 = pk2(hz, hz);
    const int y = P.target[row];
    const int vy = (y >= 0 && y < V) ? y / EPV : -1;
    const int ye = (vy >= 0) ? y - vy * EPV : 0;
    char* drow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
    for (int base = 0; base < nvec; base += kL2Threads * kL2Vec) {
      uint4 u[kL2Vec];
#pragma unroll
      for (int g = 0; g < kL2Vec; ++g) {
        const int vec = base + g * kL2Threads + tid;
        u[g] = vec < nvec ? ld_hint(zrow + int64_t(vec) * 16, drop) : Pk<T>::neutral();
      }
#pragma unroll
      for (int g = 0; g < kL2Vec; ++g) {
        const int vec = base + g * kL2Threads + tid;
        if (vec >= nvec) continue;
        float d[EPV];
        if (hz == 0.f)
          dz_vec<T, false>(u[g], d, nl2, av2, hz2);
        else
          dz_vec<T, true>(u[g], d, nl2, av2, hz2);
        if (vec == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e == ye) d[e] -= s_t;
        }
        if (vec == tail_vec) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e < tail_valid) Vec<T>::store1(drow, int64_t(vec) * EPV + e, d[e]);
        } else {
          st_stream(drow + int64_t(vec) * 16, Vec<T>::pack(d));
        }
      }
    }
  }
  if (tid == 0) {
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

// threads per CTA (TG_L2_THREADS = 256 / 512 / 1024); CTAs per SM = 1024 / threads
int l2_threads() {
  const char* e = getenv("TG_L2_THREADS");
  const int t = e ? atoi(e) : 1024;
  return (t == 256 || t == 512) ? t : 1024;
}

cudaError_t launch_fused_l2(const KParams& P, const void* meta, int n_ctas, int prefetch,
                            cudaStream_t st) {
  const RowMeta* m = reinterpret_cast<const RowMeta*>(meta);
  const bool b16 = P.dtype == TG_DTYPE_BF16;
  switch (l2_threads()) {
    case 256:
      if (b16) k_fused_l2<bf16_t, 256><<<n_ctas, 256, 0, st>>>(P, m, prefetch);
      else k_fused_l2<float, 256><<<n_ctas, 256, 0, st>>>(P, m, prefetch);
      break;
    case 512:
      if (b16) k_fused_l2<bf16_t, 512><<<n_ctas, 512, 0, st>>>(P, m, prefetch);
      else k_fused_l2<float, 512><<<n_ctas, 512, 0, st>>>(P, m, prefetch);
      break;
    default:
      if (b16) k_fused_l2<bf16_t, 1024><<<n_ctas, 1024, 0, st>>>(P, m, prefetch);
      else k_fused_l2<float, 1024><<<n_ctas, 1024, 0, st>>>(P, m, prefetch);
  }
  return cudaGetLastError();
}

}  // namespace tg
