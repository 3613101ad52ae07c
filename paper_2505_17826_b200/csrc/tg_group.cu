// tg_group.cu -- per-sequence / per-group work around the row kernels.
//
//  k_counts     batch-wide RL row / sequence counts (token-mean denominators)
//               and group-shape validation (pairwise K >= 2, DPO K == 2)
//  k_prep       K2: group-relative advantage + aggregation weight per sequence,
//               a warp-per-group segmented reduction (lanes stride over the
//               group's sequences, f64 butterfly sums -- the same bits on every
//               lane and every run; f64 like the reference's Python floats):
//                 OPMD   (r - rbar) / (1 + tau)            algorithms.py:234-242
//                 GRPO   (r - mean) / (std + eps)          north_star
//                 RLOO   r_i - mean_{j != i} r_j           north_star
//  k_rowmeta    per-row metadata (target, sequence, A, w, old / ref logprob,
//               flags) so the hot kernels have no dependent loads
//  k_seq_reduce per-sequence LP_i = sum of lp (experience_logprob,
//               algorithms.py:81-85) and the resolved reference logprob
//               (records.py:119-121 default)
//  k_coupled    K3: group-coupled coefficients of OPMD_KIMI (algorithms.py:139-146),
//               OPMD_PAIRWISE (172-183) and DPO (299-308), warp per group
//  k_finalize   deterministic fixed-order reduction of the per-CTA partial
//               stats + group metrics (combine_reports, algorithms.py:368-379)
#include <math.h>

#include "tg_common.cuh"
#include "tg_rowcoef.cuh"

namespace tg {

__device__ __forceinline__ bool is_rl(const KParams& P, int i) {
  return P.seq_kind == nullptr || P.seq_kind[i] == 0;
}

__global__ void k_counts(const KParams P) {
  __shared__ unsigned long long c[4];
  if (threadIdx.x < 4) c[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long rl_rows = 0, rl_seqs = 0, sft = 0, bad = 0;
  for (int i = threadIdx.x; i < P.n_seqs; i += blockDim.x) {
    const int n = P.seq_off[i + 1] - P.seq_off[i];
    if (n < 0) ++bad;
    if (is_rl(P, i)) {
      rl_rows += n > 0 ? n : 0;
      ++rl_seqs;
    } else {
      ++sft;
    }
  }
  for (int g = threadIdx.x; g < P.n_groups; g += blockDim.x) {
    const int k = P.grp_off[g + 1] - P.grp_off[g];
    if (k < 1) ++bad;
    if (P.pg == TG_PG_OPMD_PAIRWISE && k < 2) ++bad;
    if (P.pg == TG_PG_DPO && k != 2) ++bad;
  }
  atomicAdd(&c[0], rl_rows);
  atomicAdd(&c[1], rl_seqs);
  atomicAdd(&c[2], sft);
  atomicAdd(&c[3], bad);
  __syncthreads();
  if (threadIdx.x < 4) P.counts[threadIdx.x] = int64_t(c[threadIdx.x]);
}

__device__ __forceinline__ int warp_sum_i(int v) { return __reduce_add_sync(0xffffffffu, v); }

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

// K2, warp per group: group g's advantages and aggregation weights (per
// sequence) and metrics.  All 32 lanes call it for the same g; the group's
// RL rewards are reduced with f64 butterflies (identical on every lane).
__device__ void prep_group_warp(const KParams& P, int g, int lane, int64_t n_tok, int64_t n_seq,
                                int64_t n_sft) {
  const int a = P.grp_off[g], b = P.grp_off[g + 1];
  double sum = 0.0;
  int k = 0;
  for (int i = a + lane; i < b; i += 32)
    if (is_rl(P, i)) {
      sum += double(P.reward[i]);
      ++k;
    }
  sum = warp_sum_d(sum);
  k = warp_sum_i(k);
  const double mean = k > 0 ? sum / k : 0.0;
  double var = 0.0;
  if (P.adv == TG_ADV_GRPO && k > 1) {
    for (int i = a + lane; i < b; i += 32)
      if (is_rl(P, i)) {
        const double d = double(P.reward[i]) - mean;
        var += d * d;
      }
    var = warp_sum_d(var) / double(k - 1);
  }
  const double sd = sqrt(var);
  for (int i = a + lane; i < b; i += 32) {
    const double r = double(P.reward[i]);
    double A = 0.0, w;
    const int n_i = P.seq_off[i + 1] - P.seq_off[i];
    if (is_rl(P, i)) {
      switch (P.adv) {
        case TG_ADV_OPMD: A = (1.0 / (1.0 + double(P.tau))) * (r - mean); break;
        case TG_ADV_GRPO: A = k > 1 ? (r - mean) / (sd + double(P.std_eps)) : 0.0; break;
        case TG_ADV_RLOO: A = k > 1 ? r - (sum - r) / double(k - 1) : 0.0; break;
        case TG_ADV_REINFORCE: A = r; break;
        default: A = P.advantage ? double(P.advantage[i]) : 0.0; break;
      }
      switch (P.agg) {
        case TG_AGG_TOKEN_MEAN: w = 1.0 / double(n_tok > 0 ? n_tok : 1); break;
        case TG_AGG_SEQ_MEAN_TOKEN_SUM: w = 1.0 / double(n_seq > 0 ? n_seq : 1); break;
        case TG_AGG_SEQ_MEAN_TOKEN_MEAN:
          w = 1.0 / (double(n_seq > 0 ? n_seq : 1) * double(n_i > 0 ? n_i : 1));
          break;
        case TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM: w = 1.0 / double(P.agg_norm); break;
        default: w = 1.0; break;
      }
    } else {
      w = double(P.sft_w) / double(n_sft > 0 ? n_sft : 1);
    }
    P.sA[i] = float(A);
    P.sW[i] = float(w);
    P.sK[i] = float(b - a);
    if (P.seq_adv) P.seq_adv[i] = float(A);
  }
  if (lane == 0) {
    P.gF[4 * g + 0] = mean;
    P.gF[4 * g + 1] = mean;
    P.gF[4 * g + 2] = 0.0;
    P.gF[4 * g + 3] = double(k);
  }
}

// multi-CTA form (batches beyond one CTA's 32 warps x 64 groups): warp per group
__global__ void k_prep(const KParams P) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= P.n_groups) return;
  prep_group_warp(P, g, threadIdx.x & 31, P.n_tok_g > 0 ? P.n_tok_g : P.counts[0],
                  P.n_seq_g > 0 ? P.n_seq_g : P.counts[1],
                  P.n_sft_g > 0 ? P.n_sft_g : P.counts[2]);
}

// k_counts + k_prep in one CTA (one launch instead of two on every call):
// the batch counts are reduced in shared memory, then the 32 warps take the
// groups one warp per group.
__global__ void __launch_bounds__(1024) k_counts_prep(const KParams P) {
  pdl_trigger();  // the fused kernel may start streaming (its epilogue waits for us)
  __shared__ unsigned long long c[4];
  if (threadIdx.x < 4) c[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long rl_rows = 0, rl_seqs = 0, sft = 0, bad = 0;
  for (int i = threadIdx.x; i < P.n_seqs; i += blockDim.x) {
    const int n = P.seq_off[i + 1] - P.seq_off[i];
    if (n < 0) ++bad;
    if (is_rl(P, i)) {
      rl_rows += n > 0 ? n : 0;
      ++rl_seqs;
    } else {
      ++sft;
    }
  }
  for (int g = threadIdx.x; g < P.n_groups; g += blockDim.x) {
    const int k = P.grp_off[g + 1] - P.grp_off[g];
    if (k < 1) ++bad;
    if (P.pg == TG_PG_OPMD_PAIRWISE && k < 2) ++bad;
    if (P.pg == TG_PG_DPO && k != 2) ++bad;
  }
  if (rl_rows) atomicAdd(&c[0], rl_rows);
  if (rl_seqs) atomicAdd(&c[1], rl_seqs);
  if (sft) atomicAdd(&c[2], sft);
  if (bad) atomicAdd(&c[3], bad);
  __syncthreads();
  if (threadIdx.x < 4) P.counts[threadIdx.x] = int64_t(c[threadIdx.x]);
  const int64_t n_tok = P.n_tok_g > 0 ? P.n_tok_g : int64_t(c[0]);
  const int64_t n_seq = P.n_seq_g > 0 ? P.n_seq_g : int64_t(c[1]);
  const int64_t n_sft = P.n_sft_g > 0 ? P.n_sft_g : int64_t(c[2]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g = warp; g < P.n_groups; g += blockDim.x >> 5)
    prep_group_warp(P, g, lane, n_tok, n_seq, n_sft);
}

// one warp per sequence
__global__ void k_rowmeta(const KParams P, RowMeta* __restrict__ meta) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= P.n_seqs) return;
  const int a = P.seq_off[i], b = P.seq_off[i + 1];
  const bool rl = is_rl(P, i);
  const float A = P.sA[i], w = P.sW[i];
  const float ca = P.anchor_beta > 0.f ? P.anchor_beta / P.sK[i] : 0.f;
  for (int r = a + lane; r < b; r += 32) {
    const int32_t y = P.target[r];
    const bool bad = (y < 0) || (int64_t(y) >= P.vocab);
    // TG_PG_GIVEN: the caller's per-row coefficient / loss ride in the A / old slots
    const bool given = P.pg == TG_PG_GIVEN;
    int4 m0 = make_int4(y, i, __float_as_int(given ? P.pg_coef[r] : A), __float_as_int(w));
    int4 m1 = make_int4(__float_as_int(given ? P.pg_loss[r] : (P.old_lp ? P.old_lp[r] : 0.f)),
                        __float_as_int(P.ref_lp ? P.ref_lp[r] : 0.f),
                        int((rl ? 1u : 0u) | (bad ? 2u : 0u)), __float_as_int(ca));
    int4* dst = reinterpret_cast<int4*>(meta + r);
    dst[0] = m0;
    dst[1] = m1;
  }
}

// one warp, sequence i: LP_i and the resolved reference logprob.  Four
// independent accumulators per lane (four loads in flight), combined in a
// fixed order: the same bits from k_seq_reduce and k_tail.
__device__ __forceinline__ void seq_sums(const KParams& P, int i, int lane) {
  const int a = P.seq_off[i], b = P.seq_off[i + 1];
  double s[4] = {0.0, 0.0, 0.0, 0.0}, so[4] = {0.0, 0.0, 0.0, 0.0};
  int r = a + lane;
  for (; r + 96 < b; r += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s[u] += double(P.lp[r + 32 * u]);
      if (P.old_lp) so[u] += double(P.old_lp[r + 32 * u]);
    }
  }
  for (int u = 0; r < b; r += 32, ++u) {
    s[u] += double(P.lp[r]);
    if (P.old_lp) so[u] += double(P.old_lp[r]);
  }
  double t = warp_sum_d((s[0] + s[1]) + (s[2] + s[3]));
  double to = warp_sum_d((so[0] + so[1]) + (so[2] + so[3]));
  if (lane == 0) {
    P.sLP[i] = t;
    P.sRef[i] = P.seq_ref_lp ? double(P.seq_ref_lp[i]) : (P.old_lp ? to : t);
    P.seq_lp[i] = float(t);
  }
}

// one warp per sequence
__global__ void k_seq_reduce(const KParams P) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i < P.n_seqs) seq_sums(P, i, threadIdx.x & 31);
}

__device__ __forceinline__ double softplus_d(double x) { return log1p(exp(-fabs(x))) + fmax(x, 0.0); }
__device__ __forceinline__ double sigmoid_d(double x) {
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

// K3, warp per group: lanes stride over the group's sequences, f64 butterflies
__global__ void k_coupled(const KParams P) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= P.n_groups) return;
  const int a = P.grp_off[g], b = P.grp_off[g + 1];
  const int k = b - a;
  const double tau = double(P.tau);
  double mean = 0.0;
  for (int i = a + lane; i < b; i += 32) mean += double(P.reward[i]);
  mean = warp_sum_d(mean);
  mean = k > 0 ? mean / k : 0.0;
  double loss = 0.0, baseline = mean, aux = double(k);
  if (P.pg == TG_PG_OPMD_KIMI && k > 0) {
    double m = -INFINITY;
    for (int i = a + lane; i < b; i += 32) m = fmax(m, double(P.reward[i]));
    m = warp_max_d(m);
    double me = 0.0;
    for (int i = a + lane; i < b; i += 32) me += exp((double(P.reward[i]) - m) / tau);
    me = warp_sum_d(me);
    const double zhat = m + tau * log(me / k);  // tau_log_zhat, algorithms.py:93-101
    baseline = zhat;
    for (int i = a + lane; i < b; i += 32) {
      const double res = double(P.reward[i]) - zhat - tau * (P.sLP[i] - P.sRef[i]);
      loss += res * res;
      P.sA[i] = float(2.0 * tau * res);
    }
    loss = warp_sum_d(loss);
  } else if (P.pg == TG_PG_OPMD_PAIRWISE && k >= 2) {
    // sum_{i<j} (a_i - a_j)^2 = k sum_i (a_i - abar)^2 (centred: no cancellation)
    double tot = 0.0;
    for (int i = a + lane; i < b; i += 32) tot += double(P.reward[i]) - tau * (P.sLP[i] - P.sRef[i]);
    tot = warp_sum_d(tot);
    const double abar = tot / double(k);
    for (int i = a + lane; i < b; i += 32) {
      const double ai = double(P.reward[i]) - tau * (P.sLP[i] - P.sRef[i]);
      loss += (ai - abar) * (ai - abar);
      P.sA[i] = float(2.0 * tau * double(k) * (ai - abar));
    }
    loss = double(k) * warp_sum_d(loss);
  } else if (P.pg == TG_PG_DPO && k == 2) {
    const double n = P.n_seq_g > 0 ? double(P.n_seq_g / 2) : double(P.n_groups);
    const double beta = double(P.dpo_beta);
    const double margin = beta * ((P.sLP[a] - P.sRef[a]) - (P.sLP[a + 1] - P.sRef[a + 1]));
    loss = softplus_d(-margin) / n;
    const double s = (1.0 - sigmoid_d(margin)) * beta / n;
    if (lane == 0) {
      P.sA[a] = float(s);
      P.sA[a + 1] = float(-s);
    }
    baseline = 0.0;
    aux = margin;
  } else {
    for (int i = a + lane; i < b; i += 32) P.sA[i] = 0.f;
  }
  __syncwarp();
  for (int i = a + lane; i < b; i += 32) {
    P.sW[i] = 1.f;
    if (P.seq_adv) P.seq_adv[i] = P.sA[i];
  }
  if (lane == 0) {
    P.gF[4 * g + 0] = mean;
    P.gF[4 * g + 1] = baseline;
    P.gF[4 * g + 2] = loss;
    P.gF[4 * g + 3] = aux;
  }
}

// fixed reduction order => deterministic stats; any block size that is a
// multiple of 64 (warps stride over the 32 stats slots)
__device__ void finalize_body(const KParams& P, int coupled) {
  __shared__ double part[TG_NSTAT];
  __shared__ double grp[8];
  __shared__ double sq[3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = blockDim.x >> 5;
  for (int j = warp; j < TG_NSTAT; j += nw) {
    double s = 0.0;
    for (int c = lane; c < P.n_partials; c += 32) s += P.partials[size_t(c) * TG_NSTAT + j];
    s = warp_sum_d(s);
    if (lane == 0) part[j] = s;
  }
  if (warp == 0) {  // group metrics
    double ng = 0, smr = 0, sbl = 0, skl = 0, sgs = 0, sloss = 0, smar = 0;
    for (int g = lane; g < P.n_groups; g += 32) {
      const int a = P.grp_off[g], b = P.grp_off[g + 1];
      int k = 0;
      double kl = 0.0;
      for (int i = a; i < b; ++i)
        if (coupled || is_rl(P, i)) {
          kl += P.sRef[i] - P.sLP[i];
          ++k;
        }
      if (k == 0) continue;
      ng += 1.0;
      smr += P.gF[4 * g + 0];
      sbl += P.gF[4 * g + 1];
      skl += kl / k;
      sgs += k;
      sloss += P.gF[4 * g + 2];
      if (P.pg == TG_PG_DPO) smar += P.gF[4 * g + 3];
    }
    ng = warp_sum_d(ng); smr = warp_sum_d(smr); sbl = warp_sum_d(sbl); skl = warp_sum_d(skl);
    sgs = warp_sum_d(sgs); sloss = warp_sum_d(sloss); smar = warp_sum_d(smar);
    if (lane == 0) {
      grp[0] = ng; grp[1] = smr; grp[2] = sbl; grp[3] = skl; grp[4] = sgs; grp[5] = sloss;
      grp[6] = smar;
    }
  }
  if (warp == 1) {  // sequence sums
    double sadv = 0, nsft = 0, rsft = 0;
    for (int i = lane; i < P.n_seqs; i += 32) {
      if (coupled || is_rl(P, i)) {
        sadv += double(P.sA[i]);
      } else {
        nsft += 1.0;
        rsft += double(P.reward[i]);
      }
    }
    sadv = warp_sum_d(sadv); nsft = warp_sum_d(nsft); rsft = warp_sum_d(rsft);
    if (lane == 0) { sq[0] = sadv; sq[1] = nsft; sq[2] = rsft; }
  }
  __syncthreads();
  if (tid == 0) {
    double* o = P.stats;
    for (int j = 0; j < TG_NSTAT; ++j) o[j] = part[j];
    if (coupled) o[TG_S_PG_LOSS] = grp[5];
    o[TG_S_N_GROUPS] = grp[0];
    o[TG_S_SUM_MEAN_REWARD] = grp[1];
    o[TG_S_SUM_BASELINE] = (P.pg == TG_PG_DPO) ? 0.0 : grp[2];
    o[TG_S_SUM_KL_ESTIMATE] = grp[3];
    o[TG_S_SUM_GROUP_SIZE] = grp[4];
    o[TG_S_SUM_DPO_MARGIN] = grp[6];
    o[TG_S_N_SEQS] = double(P.n_seqs);
    o[TG_S_SUM_ADV] = coupled ? 0.0 : sq[0];
    o[TG_S_N_SFT_SEQS] = sq[1];
    o[TG_S_SUM_SFT_REWARD] = sq[2];
    o[TG_S_INVALID] += double(P.counts[3]);
    o[TG_S_LOSS] = o[TG_S_PG_LOSS] + o[TG_S_KL_LOSS] + o[TG_S_ENTROPY_LOSS] +
                   o[TG_S_ANCHOR_LOSS] + o[TG_S_SFT_LOSS];
    if (!(fabs(o[TG_S_LOSS]) <= 1.79e308)) o[TG_S_NONFINITE] += 1.0;
  }
}

// single CTA of 256 threads
__global__ void k_finalize(const KParams P, int coupled) { finalize_body(P, coupled); }

// per-sequence sums (k_seq_reduce) + k_finalize in ONE single-CTA launch for
// the per-row routes' tail: 32 warps stride over the sequences, then the
// fixed-order reduction.  PDL-launched behind the row kernel, which it waits for.
__global__ void __launch_bounds__(1024) k_tail(const KParams P) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < P.n_seqs; i += 32) seq_sums(P, i, lane);
  __syncthreads();
  finalize_body(P, 0);
}

// ---------------------------------------------------------------------------

// counts + group prep: one CTA for batches of up to 2,048 groups (every
// realistic micro-batch), two kernels beyond
int launch_group_prep(const KParams& P, bool coupled, cudaStream_t st) {
  (void)coupled;  // coupled variants get neutral per-sequence values now, A after the forward
  if (P.n_groups <= 2048) {  // <= 64 groups per warp of the single CTA
    k_counts_prep<<<1, 1024, 0, st>>>(P);
    return 1;
  }
  k_counts<<<1, 256, 0, st>>>(P);
  k_prep<<<(P.n_groups + 7) / 8, 256, 0, st>>>(P);
  return 2;
}

void launch_rowmeta(const KParams& P, void* meta, cudaStream_t st) {
  if (P.n_seqs > 0)
    k_rowmeta<<<(P.n_seqs + 7) / 8, 256, 0, st>>>(P, reinterpret_cast<RowMeta*>(meta));
}

void launch_seq_reduce(const KParams& P, cudaStream_t st) {
  if (P.n_seqs > 0) k_seq_reduce<<<(P.n_seqs + 7) / 8, 256, 0, st>>>(P);
}

void launch_coupled(const KParams& P, cudaStream_t st) {
  if (P.n_groups > 0) k_coupled<<<(P.n_groups + 7) / 8, 256, 0, st>>>(P);
}

void launch_finalize(const KParams& P, bool coupled, cudaStream_t st) {
  k_finalize<<<1, 256, 0, st>>>(P, coupled ? 1 : 0);
}

// the per-row routes' tail (seq sums + finalize) as one PDL launch; beyond
// kTailMaxRows rows the multi-CTA k_seq_reduce is faster, so two launches.
// Returns the number of kernels launched.
int launch_tail(const KParams& P, cudaStream_t st) {
  constexpr int64_t kTailMaxRows = int64_t(1) << 18;
  if (P.n_rows > kTailMaxRows) {
    launch_seq_reduce(P, st);
    launch_finalize(P, false, st);
    return (P.n_seqs > 0 ? 1 : 0) + 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_tail, P);
  return 1;
}

}  // namespace tg
