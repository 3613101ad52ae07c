// tg_stream.cu -- the two-pass route: streaming forward (K5 / K6), per-row
// coefficients, streaming backward.
//
// Used where one fused pass cannot apply:
//  * sequence-coupled losses (OPMD_KIMI algorithms.py:118-153, OPMD_PAIRWISE
//    :156-190, DPO :277-315): a row's coefficient needs its whole sequence's
//    logprob LP_i (and the group's), so the forward must finish first;
//  * the anchor KL regularizer_g (algorithms.py:193-217), which reads a second
//    logits row (the frozen anchor);
//  * tg_logprob_fwd: experience_logprob for old / ref logprob recompute
//    (algorithms.py:81-85) -- forward only, 2V bytes per row;
//  * inputs that do not meet the fused kernel's TMA alignment (any V, any
//    pitch: scalar variants).
// HBM bytes per row: forward 2V (4V with anchor), backward 4V (6V with anchor).
#include "tg_common.cuh"
#include "tg_rowcoef.cuh"
#include "tg_vecmath.cuh"

namespace tg {

constexpr int kStreamThreads = 256;
constexpr int kStreamWarps = kStreamThreads / 32;

struct OnlineU {  // online (max, sum e, sum e z, sum e (z - za))
  float m, s, t, u;
};

__device__ __forceinline__ OnlineU merge_u(OnlineU a, OnlineU b) {
  const float m = fmaxf(a.m, b.m);
  if (m == kNegInf) return {kNegInf, 0.f, 0.f, 0.f};
  const float fa = ex2((a.m - m) * kLog2e);
  const float fb = ex2((b.m - m) * kLog2e);
  return {m, a.s * fa + b.s * fb, a.t * fa + b.t * fb, a.u * fa + b.u * fb};
}

struct Lse2 {  // online (max, sum e) of the anchor row
  float m, s;
};

__device__ __forceinline__ Lse2 merge_q(Lse2 a, Lse2 b) {
  const float m = fmaxf(a.m, b.m);
  if (m == kNegInf) return {kNegInf, 0.f};
  return {m, a.s * ex2((a.m - m) * kLog2e) + b.s * ex2((b.m - m) * kLog2e)};
}

template <int N, bool ANCHOR>
__device__ __forceinline__ void accumulate(OnlineU& acc, Lse2& q, const float (&x)[N],
                                           const float (&za)[N]) {
  float vmax = x[0];
#pragma unroll
  for (int e = 1; e < N; ++e) vmax = fmaxf(vmax, x[e]);
  if (vmax > acc.m) {
    const float sc = ex2((acc.m - vmax) * kLog2e);
    acc.s *= sc;
    acc.t *= sc;
    acc.u *= sc;
    acc.m = vmax;
  }
  if (acc.m != kNegInf) {
    const float mL = acc.m * kLog2e;
#pragma unroll
    for (int e = 0; e < N; ++e) {
      const float xc = fmaxf(x[e], kClampLow);
      const float p = ex2(fmaf(xc, kLog2e, -mL));
      acc.s += p;
      acc.t = fmaf(p, xc, acc.t);
      if (ANCHOR) acc.u = fmaf(p, xc - fmaxf(za[e], kClampLow), acc.u);
    }
  }
  if (ANCHOR) {
    float qmax = za[0];
#pragma unroll
    for (int e = 1; e < N; ++e) qmax = fmaxf(qmax, za[e]);
    if (qmax > q.m) {
      q.s *= ex2((q.m - qmax) * kLog2e);
      q.m = qmax;
    }
    if (q.m != kNegInf) {
      const float mL = q.m * kLog2e;
#pragma unroll
      for (int e = 0; e < N; ++e) q.s += ex2(fmaf(fmaxf(za[e], kClampLow), kLog2e, -mL));
    }
  }
}

// ---------------------------------------------------------------------------
// forward: lse, lp, H per row (+ anchor lse_q and KL(p || q))

template <typename T, bool ANCHOR, bool VEC>
__global__ void __launch_bounds__(kStreamThreads) k_fwd(const KParams P) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  __shared__ float4 red[kStreamWarps];
  __shared__ float2 redq[kStreamWarps];
  __shared__ float redz[kStreamWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t NR = P.n_rows, V = P.vocab;
  for (int64_t row = blockIdx.x; row < NR; row += gridDim.x) {
    const int64_t src_row = P.row_index ? P.row_index[row] : row;
    const char* zrow = reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ;
    const char* qrow = ANCHOR ? reinterpret_cast<const char*>(P.anchor) + row * P.ld_anchor * ESZ
                              : nullptr;
    const int64_t y = P.target[row];
    OnlineU acc = {kNegInf, 0.f, 0.f, 0.f};
    Lse2 q = {kNegInf, 0.f};
    float zy = kNegInf;
    if (VEC) {
      const int64_t nvec = (V + EPV - 1) / EPV;
      const int64_t vy = (y >= 0 && y < V) ? y / EPV : -1;
      for (int64_t v = tid; v < nvec; v += kStreamThreads) {
        float x[EPV], za[EPV];
        Vec<T>::unpack(ld_stream(zrow + v * 16), x);
        if (ANCHOR) Vec<T>::unpack(ld_stream(qrow + v * 16), za);
        const int64_t col0 = v * EPV;
        if (col0 + EPV > V) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (col0 + e >= V) {
              x[e] = kNegInf;
              if (ANCHOR) za[e] = kNegInf;
            }
        }
        if (v == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (col0 + e == y) zy = x[e];
        }
        accumulate<EPV, ANCHOR>(acc, q, x, za);
      }
    } else {
      for (int64_t c = tid; c < V; c += kStreamThreads) {
        float x[1], za[1];
        x[0] = Vec<T>::load1(zrow, c);
        if (ANCHOR) za[0] = Vec<T>::load1(qrow, c);
        if (c == y) zy = x[0];
        accumulate<1, ANCHOR>(acc, q, x, za);
      }
    }
    // block reduction
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      OnlineU o = {__shfl_xor_sync(~0u, acc.m, d), __shfl_xor_sync(~0u, acc.s, d),
                   __shfl_xor_sync(~0u, acc.t, d), __shfl_xor_sync(~0u, acc.u, d)};
      acc = merge_u(acc, o);
      if (ANCHOR) q = merge_q(q, Lse2{__shfl_xor_sync(~0u, q.m, d), __shfl_xor_sync(~0u, q.s, d)});
    }
    zy = warp_max(zy);
    if (lane == 0) {
      red[warp] = make_float4(acc.m, acc.s, acc.t, acc.u);
      redq[warp] = make_float2(q.m, q.s);
      redz[warp] = zy;
    }
    __syncthreads();
    if (tid == 0) {
      OnlineU a = {kNegInf, 0.f, 0.f, 0.f};
      Lse2 b = {kNegInf, 0.f};
      float z = kNegInf;
      for (int w = 0; w < kStreamWarps; ++w) {
        a = merge_u(a, OnlineU{red[w].x, red[w].y, red[w].z, red[w].w});
        if (ANCHOR) b = merge_q(b, Lse2{redq[w].x, redq[w].y});
        z = fmaxf(z, redz[w]);
      }
      const float lse = a.m + logf(a.s);
      P.lse[row] = lse;
      P.lp[row] = z - lse;
      P.ent[row] = lse - a.t / a.s;
      if (ANCHOR) {
        const float lseq = b.m + logf(b.s);
        P.rLseQ[row] = lseq;
        P.rAkl[row] = a.u / a.s - lse + lseq;  // sum_v p_v (log p_v - log q_v)
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// per-row coefficients: dz_v = p_v (a + hz z_v - ca za_v) - s [v = y]

__device__ void block_store_stats(RowStats st, double anchor_loss, double anchor_kl,
                                  double* dst) {
  __shared__ double sm[kStreamWarps][17];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double v[17] = {st.pg,     st.kl,     st.ent,   st.sft,     st.clip,      st.dual,
                  st.sum_h,  st.sum_kl, st.ppo_kl, st.sum_lp, st.nonfinite, st.ratio,
                  st.n_rl,   st.invalid, st.n_rows, anchor_loss, anchor_kl};
#pragma unroll
  for (int i = 0; i < 17; ++i) v[i] = warp_sum_d(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 17; ++i) sm[warp][i] = v[i];
  __syncthreads();
  if (tid == 0) {
    double t[17];
    for (int i = 0; i < 17; ++i) {
      t[i] = 0.0;
      for (int w = 0; w < kStreamWarps; ++w) t[i] += sm[w][i];
    }
    RowStats r;
    r.pg = t[0]; r.kl = t[1]; r.ent = t[2]; r.sft = t[3]; r.clip = t[4]; r.dual = t[5];
    r.sum_h = t[6]; r.sum_kl = t[7]; r.ppo_kl = t[8]; r.sum_lp = t[9]; r.nonfinite = t[10];
    r.ratio = t[11]; r.n_rl = t[12]; r.invalid = t[13]; r.n_rows = t[14];
    r.store(dst);
    dst[TG_S_ANCHOR_LOSS] = t[15];
    dst[TG_S_SUM_ANCHOR_KL] = t[16];
  }
}

__global__ void __launch_bounds__(kStreamThreads)
    k_rowcoef(const KParams P, const RowMeta* __restrict__ meta, int coupled, int anchor) {
  RowStats st;
  st.zero();
  double aloss = 0.0, akl_sum = 0.0;
  for (int64_t row = int64_t(blockIdx.x) * kStreamThreads + threadIdx.x; row < P.n_rows;
       row += int64_t(gridDim.x) * kStreamThreads) {
    const RowMeta m = load_meta(meta, row);
    const float lp = P.lp[row], H = P.ent[row], lse = P.lse[row];
    RowTerms o;
    if (coupled) {
      o.s = P.sA[m.seq];
      o.h = o.l_pg = o.l_kl = o.l_ent = o.l_sft = o.kl = o.ratio = o.ppo_kl = 0.f;
      o.clipped = o.dual = 0;
      o.rl = 1;
    } else {
      o = meta_terms(P, m, lp, H);
    }
    const bool bad = (m.flags & 2u) != 0;
    if (bad) o.s = o.h = 0.f;
    float ca = 0.f, akl = 0.f, lseq = 0.f;
    if (anchor) {
      ca = bad ? 0.f : m.ca;
      akl = P.rAkl[row];
      lseq = P.rLseQ[row];
      aloss += double(ca) * double(akl);
      akl_sum += akl;
    }
    const float a = o.s + o.h * (H - lse) - (anchor ? ca * (lse - lseq + akl) : 0.f);
    P.rS[row] = o.s;
    P.rA[row] = a;
    P.rHz[row] = o.h + ca;
    P.rCa[row] = ca;
    const bool nonfin =
        !(finite_f(lse) && finite_f(lp) && finite_f(H) && finite_f(a) && finite_f(o.s));
    st.add(o, lp, H, bad, nonfin);
  }
  block_store_stats(st, aloss, akl_sum, P.partials + size_t(blockIdx.x) * TG_NSTAT);
}

// ---------------------------------------------------------------------------
// backward: elementwise from per-row scalars

template <typename T, bool ANCHOR, bool VEC>
__global__ void __launch_bounds__(kStreamThreads) k_bwd(const KParams P) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  const int tid = threadIdx.x;
  const int64_t NR = P.n_rows, V = P.vocab;
  for (int64_t row = blockIdx.x; row < NR; row += gridDim.x) {
    const int64_t src_row = P.row_index ? P.row_index[row] : row;
    const char* zrow = reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ;
    const char* qrow = ANCHOR ? reinterpret_cast<const char*>(P.anchor) + row * P.ld_anchor * ESZ
                              : nullptr;
    char* drow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
    const int64_t y = P.target[row];
    const float lseL = P.lse[row] * kLog2e;
    // TG_FLAG_UNSCALED_GRAD (coupled losses): p - e_y; the true row scale is in rS
    const bool unit = (P.flags & TG_FLAG_UNSCALED_GRAD) != 0;
    const float a = unit ? 1.f : P.rA[row], hz = unit ? 0.f : P.rHz[row];
    const float ca = unit ? 0.f : P.rCa[row], s = unit ? 1.f : P.rS[row];
    if (VEC) {
      const int64_t nvec = (V + EPV - 1) / EPV;
      const int64_t vy = (y >= 0 && y < V) ? y / EPV : -1;
      for (int64_t v = tid; v < nvec; v += kStreamThreads) {
        float x[EPV], za[EPV], d[EPV];
        Vec<T>::unpack(ld_stream(zrow + v * 16), x);
        if (ANCHOR) Vec<T>::unpack(ld_stream(qrow + v * 16), za);
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          const float xc = fmaxf(x[e], kClampLow);
          const float p = ex2(fmaf(xc, kLog2e, -lseL));
          float c = fmaf(hz, xc, a);
          if (ANCHOR) c = fmaf(-ca, fmaxf(za[e], kClampLow), c);
          d[e] = p * c;
        }
        const int64_t col0 = v * EPV;
        if (v == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (col0 + e == y) d[e] -= s;
        }
        if (col0 + EPV <= V) {
          st_stream(drow + v * 16, Vec<T>::pack(d));
        } else {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (col0 + e < V) Vec<T>::store1(drow, col0 + e, d[e]);
        }
      }
    } else {
      for (int64_t c = tid; c < V; c += kStreamThreads) {
        const float xc = fmaxf(Vec<T>::load1(zrow, c), kClampLow);
        const float p = ex2(fmaf(xc, kLog2e, -lseL));
        float k = fmaf(hz, xc, a);
        if (ANCHOR) k = fmaf(-ca, fmaxf(Vec<T>::load1(qrow, c), kClampLow), k);
        float d = p * k;
        if (c == y) d -= s;
        Vec<T>::store1(drow, c, d);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fast paths for the common case (no anchor, 16-byte aligned rows): four
// 128-bit streaming loads in flight per thread, packed fp32x2 math, the lazily
// rescaled accumulator of tg_vecmath.cuh, target logit read once per row.

constexpr int kFastVec = 4;  // vectors per thread per iteration

template <typename T>
__global__ void __launch_bounds__(kStreamThreads) k_fwd_fast(const KParams P) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  __shared__ float4 red[kStreamWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int V = int(P.vocab);
  const int nvec = (V + EPV - 1) / EPV;
  const int tail_vec = (V % EPV) ? nvec - 1 : -1;
  const int tail_valid = V - (nvec - 1) * EPV;
  for (int64_t row = blockIdx.x; row < P.n_rows; row += gridDim.x) {
    const int64_t src_row = P.row_index ? P.row_index[row] : row;
    const char* zrow = reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ;
    Acc2 acc = {kNegInf, pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f)};
    for (int base = 0; base < nvec; base += kStreamThreads * kFastVec) {
      uint4 u[kFastVec];
      bool valid[kFastVec];
#pragma unroll
      for (int g = 0; g < kFastVec; ++g) {
        const int vec = base + g * kStreamThreads + tid;
        valid[g] = vec < nvec;
        u[g] = valid[g] ? ld_stream(zrow + int64_t(vec) * 16) : Pk<T>::neutral();
      }
#pragma unroll
      for (int g = 0; g < kFastVec; ++g) {
        Pk<T>::clamp(u[g]);
        if (base + g * kStreamThreads + tid == tail_vec) Pk<T>::mask_from(u[g], tail_valid);
      }
      const float vmax = group_max<T>(u);
      if (__any_sync(0xffffffffu, vmax > acc.m + kSlack)) rescale(acc, vmax);
#pragma unroll
      for (int g = 0; g < kFastVec; ++g)
        if (valid[g]) accumulate<T>(acc, u[g]);
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
    if (tid == 0) {
      Online a = {kNegInf, 0.f, 0.f};
      for (int w = 0; w < kStreamWarps; ++w) a = online_merge(a, Online{red[w].x, red[w].y, red[w].z});
      const int y = P.target[row];
      const float zy = (y >= 0 && y < V) ? Vec<T>::load1(zrow, y) : kNegInf;
      const float lse = a.m + logf(a.s);
      P.lse[row] = lse;
      P.lp[row] = zy - lse;
      P.ent[row] = lse - a.t / a.s;
    }
    __syncthreads();
  }
}

template <typename T, bool kHasH>
__global__ void __launch_bounds__(kStreamThreads) k_bwd_fast(const KParams P) {
  constexpr int EPV = Vec<T>::N;
  constexpr int ESZ = elem_bytes<T>();
  const int tid = threadIdx.x;
  const int V = int(P.vocab);
  const int nvec = (V + EPV - 1) / EPV;
  const int tail_vec = (V % EPV) ? nvec - 1 : -1;
  const int tail_valid = V - (nvec - 1) * EPV;
  for (int64_t row = blockIdx.x; row < P.n_rows; row += gridDim.x) {
    const int64_t src_row = P.row_index ? P.row_index[row] : row;
    const char* zrow = reinterpret_cast<const char*>(P.logits) + src_row * P.ld * ESZ;
    char* drow = reinterpret_cast<char*>(P.dz) + row * P.ld_out * ESZ;
    const int y = P.target[row];
    const int vy = (y >= 0 && y < V) ? y / EPV : -1;
    const int ye = (vy >= 0) ? y - vy * EPV : 0;
    const float lseL = P.lse[row] * kLog2e;
    const bool unit = (P.flags & TG_FLAG_UNSCALED_GRAD) != 0;  // p - e_y (see k_bwd)
    const float a = unit ? 1.f : P.rA[row], hz = unit ? 0.f : P.rHz[row];
    const float s = unit ? 1.f : P.rS[row];
    const uint64_t nl2 = pk2(-lseL, -lseL), av2 = pk2(a, a), hz2 = pk2(hz, hz);
    for (int base = 0; base < nvec; base += kStreamThreads * kFastVec) {
      uint4 u[kFastVec];
#pragma unroll
      for (int g = 0; g < kFastVec; ++g) {
        const int vec = base + g * kStreamThreads + tid;
        u[g] = vec < nvec ? ld_stream(zrow + int64_t(vec) * 16) : Pk<T>::neutral();
      }
#pragma unroll
      for (int g = 0; g < kFastVec; ++g) {
        const int vec = base + g * kStreamThreads + tid;
        if (vec >= nvec) continue;
        float d[EPV];
        dz_vec<T, kHasH>(u[g], d, nl2, av2, hz2);
        if (vec == vy) {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e == ye) d[e] -= s;
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
}

// ---------------------------------------------------------------------------
// launch helpers

template <typename T>
static void launch_fwd_t(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st) {
  if (anchor) {
    if (vec) k_fwd<T, true, true><<<grid, kStreamThreads, 0, st>>>(P);
    else k_fwd<T, true, false><<<grid, kStreamThreads, 0, st>>>(P);
  } else {
    if (vec) k_fwd_fast<T><<<grid, kStreamThreads, 0, st>>>(P);
    else k_fwd<T, false, false><<<grid, kStreamThreads, 0, st>>>(P);
  }
}

// The backward's entropy coefficient is per row; the kHasH = true variant
// covers every row (hz = 0 rows just carry a zero coefficient).
template <typename T>
static void launch_bwd_t(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st) {
  if (anchor) {
    if (vec) k_bwd<T, true, true><<<grid, kStreamThreads, 0, st>>>(P);
    else k_bwd<T, true, false><<<grid, kStreamThreads, 0, st>>>(P);
  } else {
    if (vec) {
      if (P.entf != TG_ENT_NONE) k_bwd_fast<T, true><<<grid, kStreamThreads, 0, st>>>(P);
      else k_bwd_fast<T, false><<<grid, kStreamThreads, 0, st>>>(P);
    } else {
      k_bwd<T, false, false><<<grid, kStreamThreads, 0, st>>>(P);
    }
  }
}

void launch_fwd(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st) {
  if (P.dtype == TG_DTYPE_BF16) launch_fwd_t<bf16_t>(P, anchor, vec, grid, st);
  else launch_fwd_t<float>(P, anchor, vec, grid, st);
}

void launch_bwd(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st) {
  if (P.dtype == TG_DTYPE_BF16) launch_bwd_t<bf16_t>(P, anchor, vec, grid, st);
  else launch_bwd_t<float>(P, anchor, vec, grid, st);
}

void launch_rowcoef(const KParams& P, const void* meta, bool coupled, bool anchor, int grid,
                    cudaStream_t st) {
  k_rowcoef<<<grid, kStreamThreads, 0, st>>>(P, reinterpret_cast<const RowMeta*>(meta),
                                             coupled ? 1 : 0, anchor ? 1 : 0);
}

}  // namespace tg
