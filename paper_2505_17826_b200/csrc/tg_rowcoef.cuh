// tg_rowcoef.cuh -- the per-row epilogue shared by every loss kernel.
//
// After a row's (lse, lp, H) are known, every single-pass variant reduces to
//     dz_v = p_v * (s + h * ((z_v - lse) + H)) - s * [v == y]
// with s = -d loss / d lp (aggregation weight folded in) and h the entropy
// coefficient ("unified K1 row epilogue").  This file
// computes (s, h) and the row's loss / metric contributions from the
// registry configuration.  Restates, per row:
//   OPMD_SIMPLE policy gradient  algorithms.py:240-242  (s = A)
//   loss_sft                     algorithms.py:263-266  (s = 1/n)
// and the north_star PPO clip / dual clip, k1/k2/k3/abs KL, entropy bonus.
#pragma once

#include "tg_common.cuh"

namespace tg {

// fast exp (ex2.approx based, ~2 ulp at |x| <= 20): on the fused epilogue's
// latency-critical path
#define TG_EXPF __expf

struct RowTerms {
  float s, h;                     // gradient coefficients
  float l_pg, l_kl, l_ent, l_sft;  // weighted loss contributions
  float kl, ratio, ppo_kl;         // raw token metrics (RL rows)
  int clipped, dual, rl;
};

// Per-row metadata, prepared by k_rowmeta so the hot loop has no dependent loads.
struct __align__(16) RowMeta {
  int32_t y, seq;
  float A, w;
  float old, ref;   // TG_PG_GIVEN: A = caller's -d l / d lp, old = caller's l
  uint32_t flags;  // bit0: RL row, bit1: target outside [0, V)
  float ca;        // anchor KL coefficient beta / K of the row's group (0 = none)
};


__device__ __forceinline__ RowMeta load_meta(const RowMeta* m, int64_t row) {
  const int4* p = reinterpret_cast<const int4*>(m + row);
  int4 a = __ldg(p), b = __ldg(p + 1);
  RowMeta r;
  r.y = a.x;
  r.seq = a.y;
  r.A = __int_as_float(a.z);
  r.w = __int_as_float(a.w);
  r.old = __int_as_float(b.x);
  r.ref = __int_as_float(b.y);
  r.flags = uint32_t(b.z);
  r.ca = __int_as_float(b.w);
  return r;
}

// row_terms variant fed from RowMeta (no global loads)
__device__ __forceinline__ RowTerms meta_terms(const KParams& P, const RowMeta& m, float lp,
                                               float H) {
  RowTerms o;
  o.s = o.h = o.l_pg = o.l_kl = o.l_ent = o.l_sft = o.kl = o.ratio = o.ppo_kl = 0.f;
  o.clipped = o.dual = 0;
  o.rl = m.flags & 1u;
  if (!o.rl) {
    o.s = m.w;
    o.l_sft = -m.w * lp;
    return o;
  }
  const float A = m.A, w = m.w;
  float pg, s_pg;
  if (P.pg == TG_PG_PPO_CLIP) {
    const float old = P.old_lp ? m.old : lp;
    const float dlr = lp - old;
    const float logr = fminf(fmaxf(dlr, -20.f), 20.f);
    const float rho = TG_EXPF(logr);
    const float l1 = -A * rho;
    const float l2 = -A * fminf(fmaxf(rho, 1.f - P.clip_lo), 1.f + P.clip_hi);
    pg = fmaxf(l1, l2);
    const bool clipped = l2 > l1;
    // the log-ratio clamp is a torch.clamp: no gradient through a clamped ratio
    s_pg = (clipped || logr != dlr) ? 0.f : A * rho;
    if (P.clip_c > 0.f) {
      const float l3 = -A * P.clip_c;
      const bool dual = (A < 0.f) && (l3 < pg);
      if (dual) {
        pg = l3;
        s_pg = 0.f;
      }
      o.dual = dual;
    }
    o.clipped = clipped;
    o.ratio = rho;
    o.ppo_kl = old - lp;
  } else if (P.pg == TG_PG_SFT) {
    pg = -lp;
    s_pg = 1.f;
  } else if (P.pg == TG_PG_GIVEN) {  // RowMeta carries the caller's l_t in `old`, -dl/dlp in `A`
    pg = m.old;
    s_pg = A;
  } else {
    pg = -A * lp;
    s_pg = A;
  }
  float s_kl = 0.f, klv = 0.f;
  if (P.kl != TG_KL_NONE) {
    const float ref = P.ref_lp ? m.ref : lp;
    float dkl;
    if (P.kl == TG_KL_K1) {
      klv = lp - ref;
      dkl = 1.f;
    } else if (P.kl == TG_KL_K2) {
      const float d = lp - ref;
      klv = 0.5f * d * d;
      dkl = d;
    } else if (P.kl == TG_KL_K3) {
      const float delta = ref - lp;
      const float dcl = fminf(fmaxf(delta, -20.f), 20.f);
      const float ratio = TG_EXPF(dcl);
      const float raw = ratio - dcl - 1.f;
      klv = fminf(fmaxf(raw, -10.f), 10.f);
      dkl = (delta == dcl && raw == klv) ? 1.f - ratio : 0.f;
    } else {
      const float d = lp - ref;
      klv = fabsf(d);
      dkl = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
    }
    s_kl = -P.kl_coef * dkl;
  }
  const float c_ent = (P.entf != TG_ENT_NONE) ? P.ent_coef : 0.f;
  o.s = w * (s_pg + s_kl);
  o.h = c_ent * w;
  o.l_pg = w * pg;
  o.l_kl = w * P.kl_coef * klv;
  o.l_ent = -c_ent * w * H;
  o.kl = klv;
  return o;
}


// Per-CTA running sums of the row-level statistics, in double.
struct RowStats {
  double pg, kl, ent, sft, clip, dual, sum_h, sum_kl, ppo_kl, sum_lp, nonfinite, ratio, n_rl,
      invalid, n_rows;

  __device__ __forceinline__ void zero() {
    pg = kl = ent = sft = clip = dual = sum_h = sum_kl = ppo_kl = sum_lp = nonfinite = ratio =
        n_rl = invalid = n_rows = 0.0;
  }

  __device__ __forceinline__ void add(const RowTerms& o, float lp, float H, bool bad_target,
                                      bool nonfin) {
    pg += o.l_pg;
    kl += o.l_kl;
    ent += o.l_ent;
    sft += o.l_sft;
    clip += o.clipped;
    dual += o.dual;
    if (o.rl) {
      sum_h += H;
      sum_kl += o.kl;
      ppo_kl += o.ppo_kl;
      ratio += o.ratio;
      n_rl += 1.0;
    }
    sum_lp += lp;
    nonfinite += nonfin;
    invalid += bad_target;
    n_rows += 1.0;
  }

  __device__ __forceinline__ void merge(const RowStats& b) {
    pg += b.pg; kl += b.kl; ent += b.ent; sft += b.sft; clip += b.clip; dual += b.dual;
    sum_h += b.sum_h; sum_kl += b.sum_kl; ppo_kl += b.ppo_kl; sum_lp += b.sum_lp;
    nonfinite += b.nonfinite; ratio += b.ratio; n_rl += b.n_rl; invalid += b.invalid;
    n_rows += b.n_rows;
  }

  // write into a partial-stats row (layout TG_S_*); other slots zeroed
  __device__ __forceinline__ void store(double* dst) const {
    for (int i = 0; i < TG_NSTAT; ++i) dst[i] = 0.0;
    dst[TG_S_PG_LOSS] = pg;
    dst[TG_S_KL_LOSS] = kl;
    dst[TG_S_ENTROPY_LOSS] = ent;
    dst[TG_S_SFT_LOSS] = sft;
    dst[TG_S_CLIP_COUNT] = clip;
    dst[TG_S_DUAL_CLIP_COUNT] = dual;
    dst[TG_S_SUM_ENTROPY] = sum_h;
    dst[TG_S_SUM_KL] = sum_kl;
    dst[TG_S_SUM_PPO_KL] = ppo_kl;
    dst[TG_S_SUM_LP] = sum_lp;
    dst[TG_S_NONFINITE] = nonfinite;
    dst[TG_S_SUM_RATIO] = ratio;
    dst[TG_S_N_TOK_RL] = n_rl;
    dst[TG_S_INVALID] = invalid;
    dst[TG_S_N_TOK] = n_rows;
  }
};

__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }

}  // namespace tg
