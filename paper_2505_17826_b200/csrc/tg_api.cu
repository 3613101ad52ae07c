// tg_api.cu -- extern "C" entry points of libtg_loss.so (include/tg_loss.h).
//
// Host-side validation mirrors the reference's error behaviour
// (AlgorithmConfig.__post_init__ algorithms.py:44-56, loss-specific checks
// algorithms.py:129-135, 164-167, 232-233, 286-289), then the launch plan:
//
//   route 1 (single-pass losses, TMA-eligible input):
//       k_counts, k_prep -> k_rowmeta -> k_fused_tma -> k_seq_reduce -> k_finalize
//   route 2 (anchor KL, unaligned input, forced):
//       k_counts, k_prep -> k_rowmeta -> k_fwd -> k_rowcoef -> k_bwd -> k_seq_reduce -> k_finalize
//   route 3 (sequence-coupled OPMD_KIMI / OPMD_PAIRWISE / DPO):
//       k_counts, k_prep -> k_rowmeta -> k_fwd -> k_seq_reduce -> k_coupled -> k_rowcoef
//       -> k_bwd -> k_finalize
//
// Everything is enqueued on the caller's stream; nothing synchronises.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>

#include "tg_common.cuh"

namespace tg {
size_t fused_smem_bytes(int n_slots);
cudaError_t launch_fused(const KParams& P, const void* meta, int cl, int amode, int n_slots,
                         int n_ctas, int prefetch_rows, cudaStream_t stream);
int fused_chunk_bytes();
cudaError_t launch_lmhead_logprob(const void* hidden, int64_t ld_hidden, const void* weight,
                                  int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                                  const int32_t* target, float* lp, float* ent, float* lse,
                                  void* workspace, size_t workspace_bytes, int n_sms,
                                  cudaStream_t stream);
size_t lm_workspace_bytes(int64_t n_rows, int64_t vocab, int n_sms);
cudaError_t launch_lmhead_dz(const void* hidden, int64_t ld_hidden, const void* weight,
                             int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                             int64_t col0, int64_t n_cols, const int32_t* target,
                             const float* lse, const float* coef, void* dz, int64_t ld_dz,
                             int n_sms, cudaStream_t stream);
cudaError_t launch_update(float* table, int64_t ld_table, int64_t n_states, int64_t vocab,
                          const void* grad, int dtype, int64_t ld_grad, const int64_t* state_ids,
                          const int64_t* state_offsets, const int64_t* row_order,
                          int64_t n_touched, int64_t n_rows, double lr, int32_t* status,
                          cudaStream_t stream);
int lm_split(int64_t n_rows, int64_t vocab, int n_sms);
cudaError_t launch_grad_hidden(const void* dz, int64_t ld_dz, const void* weight,
                               int64_t ld_weight, int64_t n_rows, int64_t n_cols, int64_t dim,
                               int64_t col0, float* d_hidden, int64_t ld_dh, int accumulate,
                               int n_sms, cudaStream_t stream);
cudaError_t launch_grad_weight(const void* dz, int64_t ld_dz, const void* hidden,
                               int64_t ld_hidden, int64_t n_rows, int64_t n_cols, int64_t dim,
                               void* d_weight, int64_t ld_dw, int n_sms, cudaStream_t stream);
cudaError_t launch_grad_chunk(const void* dz, int64_t ld_dz, const void* hidden,
                              int64_t ld_hidden, const void* weight, int64_t ld_weight,
                              int64_t n_rows, int64_t n_cols, int64_t dim, int64_t col0,
                              float* d_hidden, int64_t ld_dh, int accumulate, void* d_weight,
                              int64_t ld_dw, int n_sms, cudaStream_t stream);
#ifdef TG_AB_SWITCHES
cudaError_t launch_fused_l2(const KParams& P, const void* meta, int n_ctas, int prefetch,
                            cudaStream_t st);
int l2_threads();
#endif
int fused_max_clusters(int dtype, int cl);
int fused_max_slots();
int fused_resident_chunks();
int fused_resident_chunks_z();
int fused_resident_chunks_split();
cudaError_t launch_adamw(void* param, int pdtype, int64_t ld_param, const void* grad, int gdtype,
                         int64_t ld_grad, float* m, float* v, int64_t rows, int64_t cols,
                         double lr, double b1, double b2, double eps, double wd, int64_t step,
                         int32_t* status, int n_sms, cudaStream_t st, int* n_launches);
int fused_anchor_half_bytes(int amode);
size_t rowmeta_bytes();
void launch_fwd(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st);
cudaError_t launch_fwd_tma(const KParams& P, int n_sms, cudaStream_t stream);
size_t fwd_tma_smem_bytes();
void launch_bwd(const KParams& P, bool anchor, bool vec, int grid, cudaStream_t st);
void launch_rowcoef(const KParams& P, const void* meta, bool coupled, bool anchor, int grid,
                    cudaStream_t st);
int launch_group_prep(const KParams& P, bool coupled, cudaStream_t st);
void launch_rowmeta(const KParams& P, void* meta, cudaStream_t st);
void launch_seq_reduce(const KParams& P, cudaStream_t st);
void launch_coupled(const KParams& P, cudaStream_t st);
void launch_finalize(const KParams& P, bool coupled, cudaStream_t st);
int launch_tail(const KParams& P, cudaStream_t st);
}  // namespace tg

using namespace tg;

namespace {

thread_local std::string g_err;
thread_local cudaEvent_t g_ev_begin = nullptr, g_ev_end = nullptr;
std::atomic<int64_t> g_launches{0};

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

struct DevInfo {
  int sms = 0;
  int smem_optin = 0;
};

DevInfo dev_info() {
  static std::mutex mu;
  static DevInfo cache[64];
  static bool have[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!have[dev]) {
    cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&cache[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    have[dev] = true;
  }
  return cache[dev];
}

constexpr int kMaxPartials = 1024;
constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

int esz_of(int dtype) { return dtype == TG_DTYPE_BF16 ? 2 : 4; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct Layout {
  size_t meta, lp, ent, lse, rS, rA, rHz, rCa, rLseQ, rAkl, sA, sW, sK, sLP, sRef, gF, partials,
      counts, seq_lp, total;
};

Layout layout(const TgBatch* b) {
  const size_t T = size_t(b->n_rows > 0 ? b->n_rows : 0);
  const size_t B = size_t(b->n_seqs > 0 ? b->n_seqs : 0);
  const size_t G = size_t(b->n_groups > 0 ? b->n_groups : 0);
  Layout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += align_up(bytes);
    return at;
  };
  L.meta = take(T * rowmeta_bytes());
  L.lp = take(T * 4);
  L.ent = take(T * 4);
  L.lse = take(T * 4);
  L.rS = take(T * 4);
  L.rA = take(T * 4);
  L.rHz = take(T * 4);
  L.rCa = take(T * 4);
  L.rLseQ = take(T * 4);
  L.rAkl = take(T * 4);
  L.sA = take(B * 4);
  L.sW = take(B * 4);
  L.sK = take(B * 4);
  L.sLP = take(B * 8);
  L.sRef = take(B * 8);
  L.gF = take(G * 4 * 8);
  L.partials = take(size_t(kMaxPartials) * TG_NSTAT * 8);
  L.counts = take(4 * 8);
  L.seq_lp = take(B * 4);
  L.total = o + kAlign;  // slack for re-aligning an unaligned base pointer
  return L;
}

bool coupled_pg(int pg) {
  return pg == TG_PG_OPMD_KIMI || pg == TG_PG_OPMD_PAIRWISE || pg == TG_PG_DPO;
}

int validate_batch(const TgBatch* b, bool rows_given = false) {
  if (!b) return fail(TG_EINVAL, "batch is NULL");
  if (b->dtype != TG_DTYPE_BF16 && b->dtype != TG_DTYPE_F32)
    return fail(TG_EINVAL, "unknown dtype %d", b->dtype);
  if (b->n_rows < 0 || b->n_seqs < 0 || b->n_groups < 0)
    return fail(TG_EINVAL, "negative sizes (rows %lld, seqs %d, groups %d)",
                (long long)b->n_rows, b->n_seqs, b->n_groups);
  if (b->vocab < 1) return fail(TG_EINVAL, "vocab must be >= 1, got %lld", (long long)b->vocab);
  if (b->ld < b->vocab)
    return fail(TG_EINVAL, "ld %lld < vocab %lld", (long long)b->ld, (long long)b->vocab);
  if (b->n_rows > 0 && ((!b->logits && !rows_given) || !b->target))
    return fail(TG_EINVAL, "logits and target are required when n_rows > 0");
  if (!b->seq_offsets) return fail(TG_EINVAL, "seq_offsets is required");
  if (b->n_groups > 0 && !b->group_offsets) return fail(TG_EINVAL, "group_offsets is required");
  if (b->n_seqs > 0 && !b->reward) return fail(TG_EINVAL, "reward is required");
  if (b->anchor_logits && b->ld_anchor < b->vocab)
    return fail(TG_EINVAL, "ld_anchor %lld < vocab", (long long)b->ld_anchor);
  return TG_OK;
}

int validate_cfg(const TgBatch* b, const TgConfig* c) {
  if (!c) return fail(TG_EINVAL, "config is NULL");
  if (c->advantage_fn < TG_ADV_GIVEN || c->advantage_fn > TG_ADV_REINFORCE)
    return fail(TG_EINVAL, "unknown advantage_fn %d", c->advantage_fn);
  if (c->policy_loss_fn < TG_PG_VANILLA || c->policy_loss_fn > TG_PG_GIVEN)
    return fail(TG_EINVAL, "unknown policy_loss_fn %d", c->policy_loss_fn);
  if (c->kl_fn < TG_KL_NONE || c->kl_fn > TG_KL_ABS)
    return fail(TG_EINVAL, "unknown kl_fn %d", c->kl_fn);
  if (c->entropy_loss_fn != TG_ENT_NONE && c->entropy_loss_fn != TG_ENT_DEFAULT)
    return fail(TG_EINVAL, "unknown entropy_loss_fn %d", c->entropy_loss_fn);
  if (c->loss_agg_mode < TG_AGG_SEQ_SUM || c->loss_agg_mode > TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM)
    return fail(TG_EINVAL, "unknown loss_agg_mode %d", c->loss_agg_mode);
  if (!(c->tau >= 0)) return fail(TG_EINVAL, "tau must be >= 0, got %g", c->tau);
  if ((c->policy_loss_fn == TG_PG_OPMD_KIMI || c->policy_loss_fn == TG_PG_OPMD_PAIRWISE) &&
      !(c->tau > 0))
    return fail(TG_EINVAL, "%s requires tau > 0",
                c->policy_loss_fn == TG_PG_OPMD_KIMI ? "OPMD_KIMI" : "OPMD_PAIRWISE");
  if (!(c->anchor_beta >= 0)) return fail(TG_EINVAL, "beta must be >= 0, got %g", c->anchor_beta);
  if (c->anchor_beta > 0 && !b->anchor_logits)
    return fail(TG_EINVAL, "beta > 0 requires sft_params (anchor_logits)");
  if (!(c->dpo_beta > 0)) return fail(TG_EINVAL, "dpo_beta must be > 0, got %g", c->dpo_beta);
  if (!(c->clip_lo >= 0) || !(c->clip_hi >= 0))
    return fail(TG_EINVAL, "clip ranges must be >= 0");
  if (c->clip_c != 0 && !(c->clip_c > 1)) return fail(TG_EINVAL, "clip_c must be 0 or > 1");
  if (!(c->std_eps >= 0)) return fail(TG_EINVAL, "std_eps must be >= 0");
  if (!(c->sft_weight >= 0)) return fail(TG_EINVAL, "sft_weight must be >= 0");
  if (c->loss_agg_mode == TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM && !(c->agg_norm > 0))
    return fail(TG_EINVAL, "agg_norm must be > 0");
  if (coupled_pg(c->policy_loss_fn)) {
    // whole-sequence objectives: no per-token penalty, bonus, aggregation or SFT rows
    if (c->kl_fn != TG_KL_NONE && c->kl_coef != 0)
      return fail(TG_EINVAL, "sequence-coupled losses take no token KL penalty");
    if (c->entropy_loss_fn != TG_ENT_NONE && c->entropy_coef != 0)
      return fail(TG_EINVAL, "sequence-coupled losses take no entropy bonus");
    if (c->loss_agg_mode != TG_AGG_SEQ_SUM)
      return fail(TG_EINVAL, "sequence-coupled losses sum over groups (loss_agg_mode SEQ_SUM)");
    if (b->seq_kind || c->n_sft_seq_global > 0)
      return fail(TG_EINVAL, "sequence-coupled losses take no SFT rows (seq_kind must be NULL)");
  }
  if (c->policy_loss_fn == TG_PG_GIVEN && b->n_rows > 0 && (!b->pg_coef || !b->pg_loss))
    return fail(TG_EINVAL, "policy_loss_fn GIVEN requires batch.pg_coef and batch.pg_loss");
  if (c->advantage_fn == TG_ADV_GIVEN &&
      (c->policy_loss_fn == TG_PG_VANILLA || c->policy_loss_fn == TG_PG_PPO_CLIP) &&
      b->n_seqs > 0 && !b->advantage)
    return fail(TG_EINVAL, "advantage_fn GIVEN requires batch.advantage");
  return TG_OK;
}

void fill_params(KParams& P, const TgBatch* b, const TgConfig* c, const TgOut* o, char* ws,
                 const Layout& L) {
  memset(&P, 0, sizeof(P));
  P.logits = b->logits;
  P.row_index = b->row_index;
  P.anchor = b->anchor_logits;
  P.n_rows = b->n_rows;
  P.vocab = b->vocab;
  P.ld = b->ld;
  P.ld_anchor = b->ld_anchor;
  P.ld_out = (o && o->dlogits) ? o->ld_out : b->ld;
  P.dtype = b->dtype;
  P.n_seqs = b->n_seqs;
  P.n_groups = b->n_groups;
  P.target = b->target;
  P.old_lp = b->old_lp;
  P.ref_lp = b->ref_lp;
  P.seq_off = b->seq_offsets;
  P.grp_off = b->group_offsets;
  P.reward = b->reward;
  P.seq_ref_lp = b->seq_ref_lp;
  P.advantage = b->advantage;
  P.seq_kind = b->seq_kind;
  P.pg_coef = b->pg_coef;
  P.pg_loss = b->pg_loss;
  P.dz = o ? o->dlogits : nullptr;
  P.lp = (o && o->lp) ? o->lp : reinterpret_cast<float*>(ws + L.lp);
  P.ent = (o && o->entropy) ? o->entropy : reinterpret_cast<float*>(ws + L.ent);
  P.lse = (o && o->lse) ? o->lse : reinterpret_cast<float*>(ws + L.lse);
  P.seq_lp = (o && o->seq_lp) ? o->seq_lp : reinterpret_cast<float*>(ws + L.seq_lp);
  P.seq_adv = o ? o->seq_adv : nullptr;
  P.stats = o ? o->stats : nullptr;
  P.sA = reinterpret_cast<float*>(ws + L.sA);
  P.sW = reinterpret_cast<float*>(ws + L.sW);
  P.sK = reinterpret_cast<float*>(ws + L.sK);
  P.sLP = reinterpret_cast<double*>(ws + L.sLP);
  P.sRef = reinterpret_cast<double*>(ws + L.sRef);
  P.gF = reinterpret_cast<double*>(ws + L.gF);
  if (o && o->row_coef) {  // caller-visible row coefficients [3, T]: a, hz, s
    P.rA = o->row_coef;
    P.rHz = o->row_coef + b->n_rows;
    P.rS = o->row_coef + 2 * b->n_rows;
  } else {
    P.rS = reinterpret_cast<float*>(ws + L.rS);
    P.rA = reinterpret_cast<float*>(ws + L.rA);
    P.rHz = reinterpret_cast<float*>(ws + L.rHz);
  }
  P.rCa = reinterpret_cast<float*>(ws + L.rCa);
  P.rLseQ = reinterpret_cast<float*>(ws + L.rLseQ);
  P.rAkl = reinterpret_cast<float*>(ws + L.rAkl);
  P.partials = reinterpret_cast<double*>(ws + L.partials);
  P.counts = reinterpret_cast<int64_t*>(ws + L.counts);
  if (c) {
    P.adv = c->advantage_fn;
    P.pg = c->policy_loss_fn;
    P.kl = c->kl_fn;
    P.entf = c->entropy_loss_fn;
    P.agg = c->loss_agg_mode;
    P.flags = c->flags;
    P.tau = float(c->tau);
    P.clip_lo = float(c->clip_lo);
    P.clip_hi = float(c->clip_hi);
    P.clip_c = float(c->clip_c);
    P.kl_coef = float(c->kl_coef);
    P.ent_coef = float(c->entropy_coef);
    P.std_eps = float(c->std_eps);
    P.sft_w = float(c->sft_weight);
    P.anchor_beta = float(c->anchor_beta);
    P.dpo_beta = float(c->dpo_beta);
    P.agg_norm = float(c->agg_norm);
    P.n_tok_g = c->n_tok_global;
    P.n_seq_g = c->n_seq_global;
    P.n_sft_g = c->n_sft_seq_global;
  }
}

// Fused-kernel plan: cluster size and ring slots, or cl = 0 if not eligible.
struct FusedPlan {
  int cl = 0, n_slots = 0, n_ctas = 0, prefetch_rows = 1;
  // anchor KL: 1 = z + za stashed in TMEM, 2 = z stashed, za re-read from L2,
  // 3 = z + za stashed in TMEM and shared-memory positions
  int amode = 0;
};

// Tuning overrides for measurement, A/B build only (tg_common.cuh ab_env):
// TG_FUSED_CL=1|2|3|4 forces the cluster size, TG_PREFETCH_ROWS=n the L2
// look-ahead depth (rows per cluster; 0 disables).
int env_int(const char* name, int dflt) { return ab_env(name, dflt); }

FusedPlan fused_plan(const TgBatch* b, const TgOut* o, bool anchor = false) {
  FusedPlan fp;
  // L2 look-ahead measured neutral at 1 row and harmful beyond (extra DRAM
  // reads from prefetched lines evicted before use): off by default
  fp.prefetch_rows = env_int("TG_PREFETCH_ROWS", 0);
  const int force_cl = env_int("TG_FUSED_CL", 0);
  const int esz = esz_of(b->dtype);
  const int epv = 16 / esz;
  if (!o || !o->dlogits) return fp;
  if (!aligned16(b->logits) || (b->ld * esz) % 16 != 0) return fp;
  if (!aligned16(o->dlogits) || (o->ld_out * esz) % 16 != 0 || o->ld_out < b->vocab) return fp;
  const int64_t nvec = (b->vocab + epv - 1) / epv;
  if (b->ld < nvec * epv) return fp;  // TMA reads whole 16-byte vectors
  if (anchor) {  // the anchor rows ride the same ring: aligned, whole vectors
    if (!aligned16(b->anchor_logits) ||
        (b->ld_anchor * esz) % 16 != 0 || b->ld_anchor < nvec * epv)
      return fp;
    if (env_int("TG_FUSED_ANCHOR", 1) == 0) return fp;
  }
  const DevInfo d = dev_info();
  if (d.sms <= 0) return fp;
  const size_t tail = fused_smem_bytes(0);
  int n_slots = int((size_t(d.smem_optin) - tail) / size_t(fused_chunk_bytes()));
  if (n_slots > fused_max_slots()) n_slots = fused_max_slots();
  if (n_slots < fused_max_slots()) return fp;  // the kernel's ring size is compile-time
  static const int kOrder[4] = {1, 2, 4, 3};
  // anchor KL: mode 1 (z and za stashed) at the smallest cluster size that
  // holds both slices, else mode 2 (z stashed, za re-read from L2 in phase 2:
  // twice the columns per CTA).  Mode 2 where mode 1 also fits measured slower
  // (profiles/r02_anchor_modes.txt: 4.63 vs 4.99 TB/s at V = 151,936 bf16,
  // CL = 2 vs 4 -- the L2 re-read stalls phase 2 and 7 % of it misses), so it
  // only serves rows neither mode 1 nor mode 3 holds (e.g. bf16 rows of ~200 k
  // columns: still 6V bytes instead of the two-pass 10V).  TG_FUSED_ANCHOR_MODE
  // forces one (A/B build).
  //
  // Mode 3 (split stash: 8 TMEM + 5 shared-memory z + za pair positions) holds
  // a 2-CTA slice at V = 151,936 bf16, so those rows run on 2-CTA clusters over
  // all 148 SMs instead of mode 1's 4-CTA clusters on 132 (5.29 vs 4.99 TB/s),
  // and fp32 rows at that vocabulary on 4-CTA clusters (5.93 vs 5.17 TB/s for
  // mode 2; profiles/r02_anchor_split.txt).  Per cluster size the order is
  // mode 1, mode 3 (pass 0), then mode 2 (pass 1).
  const int force_mode = anchor ? env_int("TG_FUSED_ANCHOR_MODE", 0) : 0;
  static const int kModeOrder[2][2] = {{1, 3}, {2, 0}};
  const int n_pass = anchor ? (force_mode ? 1 : 2) : 1;
  for (int pass = 0; pass < n_pass; ++pass)
  for (int oi = 0; oi < 4; ++oi) {
    const int cl = kOrder[oi];
    if (force_cl ? cl != force_cl : cl == 3) continue;  // CL = 3 only on request
    if (anchor && cl == 3 && b->dtype != TG_DTYPE_BF16) continue;  // not instantiated
    const int64_t slice_vec = (nvec + cl - 1) / cl;
    const int64_t nchunk = (slice_vec * 16 + fused_chunk_bytes() - 1) / fused_chunk_bytes();
    // resident TMEM chunks: the slice + >= 2 prefix chunks (anchor: a stash
    // slot holds a z + za half-chunk pair in modes 1 / 3, the z half chunk in mode 2)
    int amode = 0;
    int64_t need = nchunk + 2;
    if (anchor) {
      const int64_t half = fused_anchor_half_bytes(1);
      const int64_t nslot = (slice_vec * 16 + half - 1) / half;
      // (a forced cluster size may run with a single slot of look-ahead)
      need = nslot + (force_cl ? 1 : 2);
      for (int mi = 0; mi < 2 && amode == 0; ++mi) {
        const int want = force_mode ? (mi == 0 ? force_mode : 0) : kModeOrder[pass][mi];
        if (want == 1 && need <= fused_resident_chunks()) amode = 1;
        if (want == 2 && need <= fused_resident_chunks_z() &&
            (cl == 2 || (cl == 1 && b->dtype == TG_DTYPE_BF16) ||
             (cl == 4 && b->dtype != TG_DTYPE_BF16)))  // instantiated
          amode = 2;
        if (want == 3 && need <= fused_resident_chunks_split() &&
            ((cl == 2 && b->dtype == TG_DTYPE_BF16) ||
             (cl == 4 && b->dtype != TG_DTYPE_BF16)))  // instantiated
          amode = 3;
      }
    }
    if (anchor ? amode != 0 : need <= fused_resident_chunks()) {
      // persistent grid: as many clusters as can be co-resident, at most one per row
      int64_t clusters_max = fused_max_clusters(b->dtype, cl);
      if (clusters_max <= 0) clusters_max = d.sms / cl;
      const int64_t clusters = b->n_rows < clusters_max ? b->n_rows : clusters_max;
      fp.cl = cl;
      fp.amode = amode;
      // mode 3: L2 look-ahead of the stash positions behind the landing slots
      // (kernel argument bits 16..31)
      if (amode == 3) fp.prefetch_rows |= env_int("TG_PREFETCH_CHUNKS", 6) << 16;
      else fp.prefetch_rows |= env_int("TG_PREFETCH_CHUNKS", 0) << 16;  // (A/B only)
      fp.n_slots = n_slots;
      fp.n_ctas = int(clusters * cl);
      return fp;
    }
  }
  return fp;
}

// Forward pass of the two-pass / coupled routes and tg_logprob_fwd: the TMA
// streaming kernel (k_fwd_tma) for 16-byte-aligned rows without an anchor, the
// grid-stride kernels otherwise.  TG_FWD_TMA=0 forces the latter (A/B).
void run_forward(const KParams& P, const TgBatch* b, bool anchor, bool vin, int grid,
                 cudaStream_t st) {
  const int esz = esz_of(b->dtype);
  const int epv = 16 / esz;
  const int64_t nvec = (b->vocab + epv - 1) / epv;
  const DevInfo d = dev_info();
  const bool tma = !anchor && vin && env_int("TG_FWD_TMA", 1) != 0 && b->ld >= nvec * epv &&
                   d.sms > 0 && size_t(d.smem_optin) >= fwd_tma_smem_bytes();
  if (tma && launch_fwd_tma(P, d.sms, st) == cudaSuccess) return;
  cudaGetLastError();
  launch_fwd(P, anchor, vin, grid, st);
}

int route_of(const TgBatch* b, const TgConfig* c, const TgOut* o) {
  if (coupled_pg(c->policy_loss_fn)) {
    if ((c->flags & TG_FLAG_UNSCALED_GRAD) && o && o->dlogits && c->anchor_beta <= 0 &&
        !(c->flags & (TG_FLAG_FORCE_TWO_PASS | TG_FLAG_ROWS_GIVEN)) && fused_plan(b, o).cl != 0)
      return 4;
    return 3;
  }
  if (c->flags & TG_FLAG_ROWS_GIVEN) return 2;
  if (o && o->row_coef) return 2;  // the fused kernel keeps the coefficients on chip
  if (c->anchor_beta > 0)  // fused anchor KL (6V) when the layout allows, else two-pass (10V)
    return (o && o->dlogits && !(c->flags & (TG_FLAG_FORCE_TWO_PASS | TG_FLAG_NO_FUSED_TMA)) &&
            fused_plan(b, o, true).cl != 0)
               ? 1
               : 2;
  if (c->flags & (TG_FLAG_FORCE_TWO_PASS | TG_FLAG_NO_FUSED_TMA)) return 2;
  if (!o || !o->dlogits) return 2;
  if (fused_plan(b, o).cl == 0) return 2;
  return 1;
}

int stream_grid(int64_t rows) {
  const DevInfo d = dev_info();
  const int64_t cap = int64_t(d.sms > 0 ? d.sms : 148) * 8;
  return int(rows < cap ? (rows > 0 ? rows : 1) : cap);
}

bool vec_ok(const void* p, int64_t ld, int esz) {
  return aligned16(p) && (ld * esz) % 16 == 0;
}

char* align_ws(void* ws) {
  uintptr_t p = reinterpret_cast<uintptr_t>(ws);
  p = (p + kAlign - 1) / kAlign * kAlign;
  return reinterpret_cast<char*>(p);
}

int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return TG_OK;
}

}  // namespace

extern "C" {

size_t tg_workspace_size(const TgBatch* batch, const TgConfig* /*cfg*/) {
  if (!batch) return 0;
  return layout(batch).total;
}

int tg_route(const TgBatch* batch, const TgConfig* cfg) {
  if (!batch || !cfg) return 0;
  TgOut probe = {};
  probe.dlogits = const_cast<void*>(batch->logits);
  probe.ld_out = batch->ld;
  return route_of(batch, cfg, &probe);
}

int tg_fused_cluster_size(const TgBatch* batch, const TgConfig* cfg) {
  if (!batch || !cfg) return 0;
  TgOut probe = {};
  probe.dlogits = const_cast<void*>(batch->logits);
  probe.ld_out = batch->ld;
  const int r = route_of(batch, cfg, &probe);
  if (r != 1 && r != 4) return 0;
  return fused_plan(batch, &probe, r == 1 && cfg->anchor_beta > 0).cl;
}

int tg_loss_fwd_bwd(const TgBatch* b, const TgConfig* c, TgOut* o, void* workspace,
                    size_t workspace_bytes, void* stream) {
  const bool rows_given = c && (c->flags & TG_FLAG_ROWS_GIVEN);
  if (rows_given) {
    if (!o || !o->lp || !o->entropy || !o->lse)
      return fail(TG_EINVAL, "TG_FLAG_ROWS_GIVEN needs out.lp, out.entropy and out.lse (inputs)");
    if (o->dlogits) return fail(TG_EINVAL, "TG_FLAG_ROWS_GIVEN is forward-only: dlogits must be NULL");
    if (b && b->anchor_logits)
      return fail(TG_EINVAL, "TG_FLAG_ROWS_GIVEN cannot evaluate the anchor KL (needs logits)");
  }
  int rc = validate_batch(b, rows_given);
  if (rc) return rc;
  rc = validate_cfg(b, c);
  if (rc) return rc;
  if (!o || !o->stats) return fail(TG_EINVAL, "out.stats is required");
  if (c->flags & TG_FLAG_UNSCALED_GRAD) {
    if (!coupled_pg(c->policy_loss_fn))
      return fail(TG_EINVAL, "TG_FLAG_UNSCALED_GRAD applies to sequence-coupled losses "
                             "(OPMD_KIMI / OPMD_PAIRWISE / DPO) only");
    if (!o->dlogits || !o->row_coef)
      return fail(TG_EINVAL, "TG_FLAG_UNSCALED_GRAD needs out.dlogits and out.row_coef");
    if (c->flags & TG_FLAG_ROWS_GIVEN)
      return fail(TG_EINVAL, "TG_FLAG_UNSCALED_GRAD and TG_FLAG_ROWS_GIVEN exclude each other");
    if (c->anchor_beta > 0)
      return fail(TG_EINVAL, "TG_FLAG_UNSCALED_GRAD cannot describe the anchor-KL gradient");
  }
  if (o->row_coef && c->anchor_beta > 0)
    return fail(TG_EINVAL, "out.row_coef cannot describe the anchor-KL gradient (anchor_beta > 0)");
  if (o->dlogits) {
    if (o->ld_out < b->vocab) return fail(TG_EINVAL, "ld_out < vocab");
    if (o->dlogits == b->logits && (b->row_index || o->ld_out != b->ld))
      return fail(TG_EINVAL, "in-place dlogits requires ld_out == ld and no row_index");
  }
  const Layout L = layout(b);
  if (!workspace || workspace_bytes < L.total)
    return fail(TG_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", L.total,
                workspace_bytes);
  char* ws = align_ws(workspace);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  KParams P;
  fill_params(P, b, c, o, ws, L);
  void* meta = ws + L.meta;
  // TG_FLAG_UNSCALED_GRAD without a single-pass plan (pitch / dtype / forced
  // two-pass) runs route 3 with a unit-coefficient backward: same outputs, 6V bytes
  const int route = route_of(b, c, o);
  const bool coupled = route == 3 || route == 4;
  const bool anchor = c->anchor_beta > 0;
  const int esz = esz_of(b->dtype);
  cudaGetLastError();  // clear stale errors

  cudaEvent_t ev_begin = g_ev_begin, ev_end = g_ev_end;
  g_ev_begin = g_ev_end = nullptr;
  // the timing span is the whole call (prologue, row kernels, tail): events
  // between PDL-chained kernels would serialise them
  if (ev_begin) cudaEventRecord(ev_begin, st);
  count_launches(launch_group_prep(P, coupled, st));
  if (route == 4) {
    // coupled loss in one pass: the fused kernel writes p - e_y and the per-row
    // lp / entropy / lse; the sequence sums, the coupled coefficients and the
    // per-row scale (row_coef) follow as in route 3, without a backward pass
    const FusedPlan fp = fused_plan(b, o);
    P.n_partials = fp.n_ctas;
    if (P.n_partials > kMaxPartials) return fail(TG_EUNSUPPORTED, "too many CTAs");
    if (b->n_rows > 0) {
      cudaError_t e = launch_fused(P, meta, fp.cl, fp.amode, fp.n_slots, fp.n_ctas, fp.prefetch_rows, st);
      if (e != cudaSuccess) return fail(TG_ECUDA, "fused kernel launch: %s", cudaGetErrorString(e));
      count_launches(1);
    }
    launch_rowmeta(P, meta, st);
    launch_seq_reduce(P, st);
    launch_coupled(P, st);
    count_launches((b->n_seqs > 0 ? 2 : 0) + (b->n_groups > 0 ? 1 : 0));
    int cgrid = int((b->n_rows + 255) / 256);
    if (cgrid < 1) cgrid = 1;
    if (cgrid > kMaxPartials) cgrid = kMaxPartials;
    P.n_partials = cgrid;
    launch_rowcoef(P, meta, true, false, cgrid, st);
    count_launches(1);
  } else if (route == 1) {
    const FusedPlan fp = fused_plan(b, o, anchor);
#ifdef TG_AB_SWITCHES
    // TG_FUSED_IMPL=2: the L2-reread variant (tg_fused_l2.cu), A/B build only
    const bool l2 = env_int("TG_FUSED_IMPL", 0) == 2;
    const int64_t l2_slots = int64_t(dev_info().sms) * (1024 / l2_threads());
    const int l2_ctas = int(b->n_rows < l2_slots ? b->n_rows : l2_slots);
#else
    constexpr bool l2 = false;
    constexpr int l2_ctas = 0;
#endif
    P.n_partials = l2 ? l2_ctas : fp.n_ctas;
    if (P.n_partials > kMaxPartials) return fail(TG_EUNSUPPORTED, "too many CTAs");
    if (b->n_rows > 0) {
      if (l2) {  // the L2 variant reads the packed per-row metadata
        launch_rowmeta(P, meta, st);
        count_launches(b->n_seqs > 0 ? 1 : 0);
      }
#ifdef TG_AB_SWITCHES
      cudaError_t e = l2 ? launch_fused_l2(P, meta, l2_ctas, fp.prefetch_rows, st)
                         : launch_fused(P, meta, fp.cl, fp.amode, fp.n_slots, fp.n_ctas, fp.prefetch_rows, st);
#else
      cudaError_t e = launch_fused(P, meta, fp.cl, fp.amode, fp.n_slots, fp.n_ctas, fp.prefetch_rows, st);
#endif
      if (e != cudaSuccess) return fail(TG_ECUDA, "fused kernel launch: %s", cudaGetErrorString(e));
      count_launches(1);
    } else {
      P.n_partials = 0;
    }
    count_launches(launch_tail(P, st));  // seq sums + finalize
    if (ev_end) cudaEventRecord(ev_end, st);
    return check_cuda("tg_loss_fwd_bwd");
  } else {
    launch_rowmeta(P, meta, st);
    count_launches(b->n_seqs > 0 ? 1 : 0);
    const bool vin = vec_ok(b->logits, b->ld, esz) &&
                     (!anchor || vec_ok(b->anchor_logits, b->ld_anchor, esz));
    const int grid = stream_grid(b->n_rows);
    if (b->n_rows > 0 && !rows_given) {
      run_forward(P, b, anchor, vin, grid, st);
      count_launches(1);
    }
    if (coupled) {
      launch_seq_reduce(P, st);
      launch_coupled(P, st);
      count_launches((b->n_seqs > 0 ? 1 : 0) + (b->n_groups > 0 ? 1 : 0));
    }
    int cgrid = int((b->n_rows + 255) / 256);
    if (cgrid < 1) cgrid = 1;
    if (cgrid > kMaxPartials) cgrid = kMaxPartials;
    P.n_partials = cgrid;
    launch_rowcoef(P, meta, coupled, anchor, cgrid, st);
    count_launches(1);
    if (o->dlogits && b->n_rows > 0) {
      const bool vout = vin && vec_ok(o->dlogits, o->ld_out, esz);
      launch_bwd(P, anchor, vout, grid, st);
      count_launches(1);
    }
    if (!coupled) {
      count_launches(launch_tail(P, st));  // seq sums + finalize
      if (ev_end) cudaEventRecord(ev_end, st);
      return check_cuda("tg_loss_fwd_bwd");
    }
  }
  launch_finalize(P, coupled, st);
  count_launches(1);
  if (ev_end) cudaEventRecord(ev_end, st);
  return check_cuda("tg_loss_fwd_bwd");
}

int tg_logprob_fwd(const TgBatch* b, TgOut* o, void* workspace, size_t workspace_bytes,
                   void* stream) {
  int rc = validate_batch(b);
  if (rc) return rc;
  if (!o) return fail(TG_EINVAL, "out is NULL");
  const Layout L = layout(b);
  if (!workspace || workspace_bytes < L.total)
    return fail(TG_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", L.total,
                workspace_bytes);
  char* ws = align_ws(workspace);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  KParams P;
  fill_params(P, b, nullptr, o, ws, L);
  P.dz = nullptr;
  cudaGetLastError();
  const int esz = esz_of(b->dtype);
  if (b->n_rows > 0) {
    run_forward(P, b, false, vec_ok(b->logits, b->ld, esz), stream_grid(b->n_rows), st);
    count_launches(1);
  }
  if (o->seq_lp && b->n_seqs > 0) {
    launch_seq_reduce(P, st);
    count_launches(1);
  }
  return check_cuda("tg_logprob_fwd");
}

// size / pitch / alignment rules shared by the LM-head entry points
static int lmhead_check(const void* hidden, int64_t ld_hidden, const void* weight,
                        int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim) {
  if (n_rows < 0 || vocab < 1 || dim < 1)
    return fail(TG_EINVAL, "bad sizes (rows %lld, vocab %lld, dim %lld)", (long long)n_rows,
                (long long)vocab, (long long)dim);
  if (dim % 64 != 0) return fail(TG_EINVAL, "dim must be a multiple of 64, got %lld", (long long)dim);
  if (ld_hidden < dim || ld_weight < dim)
    return fail(TG_EINVAL, "row pitch below dim (ld_hidden %lld, ld_weight %lld)",
                (long long)ld_hidden, (long long)ld_weight);
  if (ld_hidden % 8 != 0 || ld_weight % 8 != 0)
    return fail(TG_EINVAL, "row pitches must be multiples of 8 elements (16 bytes)");
  if (vocab > (int64_t(1) << 31) - 256 || n_rows > (int64_t(1) << 31) - 128)
    return fail(TG_EINVAL, "vocab / rows too large");
  if (n_rows > 0 && (!hidden || !weight)) return fail(TG_EINVAL, "hidden and weight are required");
  if (n_rows > 0 && (!aligned16(hidden) || !aligned16(weight)))
    return fail(TG_EINVAL, "hidden and weight must be 16-byte aligned");
  return TG_OK;
}

int tg_lmhead_logprob_fwd(const void* hidden, int64_t ld_hidden, const void* weight,
                          int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                          const int32_t* target, float* lp, float* entropy, float* lse,
                          void* workspace, size_t workspace_bytes, void* stream) {
  const int rc = lmhead_check(hidden, ld_hidden, weight, ld_weight, n_rows, vocab, dim);
  if (rc) return rc;
  if (n_rows == 0) return TG_OK;
  if (!lse || !entropy) return fail(TG_EINVAL, "entropy and lse are required");
  if (lp && !target) return fail(TG_EINVAL, "lp requires target");
  const DevInfo d = dev_info();
  const int sms = d.sms > 0 ? d.sms : 148;
  const size_t need = lm_workspace_bytes(n_rows, vocab, sms);
  if (need > 0 && (!workspace || workspace_bytes < need))
    return fail(TG_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", need,
                workspace_bytes);
  if (need > 0 && !aligned16(workspace)) return fail(TG_EINVAL, "workspace must be 16-byte aligned");
  cudaGetLastError();
  cudaError_t e = launch_lmhead_logprob(hidden, ld_hidden, weight, ld_weight, n_rows, vocab, dim,
                                        target, lp, entropy, lse, workspace, workspace_bytes, sms,
                                        reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(TG_EUNSUPPORTED, "cuTensorMapEncodeTiled is unavailable (driver too old)");
  count_launches(lm_split(n_rows, vocab, sms) > 1 ? 2 : 1);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_lmhead_logprob_fwd: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_lmhead_dlogits(const void* hidden, int64_t ld_hidden, const void* weight,
                      int64_t ld_weight, int64_t n_rows, int64_t vocab, int64_t dim,
                      int64_t col0, int64_t n_cols, const int32_t* target, const float* lse,
                      const float* row_coef, void* dz, int64_t ld_dz, void* stream) {
  const int rc = lmhead_check(hidden, ld_hidden, weight, ld_weight, n_rows, vocab, dim);
  if (rc) return rc;
  if (col0 < 0 || n_cols < 1 || col0 + n_cols > vocab)
    return fail(TG_EINVAL, "vocabulary chunk [%lld, %lld) outside [0, %lld)", (long long)col0,
                (long long)(col0 + n_cols), (long long)vocab);
  if (ld_dz < n_cols || ld_dz % 8 != 0)
    return fail(TG_EINVAL, "ld_dz must be >= n_cols and a multiple of 8, got %lld",
                (long long)ld_dz);
  if (n_rows == 0) return TG_OK;
  if (!target || !lse || !row_coef || !dz)
    return fail(TG_EINVAL, "target, lse, row_coef and dz are required");
  if (!aligned16(dz)) return fail(TG_EINVAL, "dz must be 16-byte aligned");
  const DevInfo d = dev_info();
  const int sms = d.sms > 0 ? d.sms : 148;
  cudaGetLastError();
  cudaError_t e = launch_lmhead_dz(hidden, ld_hidden, weight, ld_weight, n_rows, vocab, dim, col0,
                                   n_cols, target, lse, row_coef, dz, ld_dz, sms,
                                   reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(TG_EUNSUPPORTED, "cuTensorMapEncodeTiled is unavailable (driver too old)");
  count_launches(1);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_lmhead_dlogits: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_lmhead_grad_hidden(const void* dz, int64_t ld_dz, const void* weight, int64_t ld_weight,
                          int64_t n_rows, int64_t vocab, int64_t dim, int64_t col0,
                          int64_t n_cols, float* d_hidden, int64_t ld_dh, int accumulate,
                          void* stream) {
  // (hidden is not read: check the weight's layout with itself in its place)
  const int rc = lmhead_check(weight, ld_weight, weight, ld_weight, n_rows, vocab, dim);
  if (rc) return rc;
  if (col0 < 0 || n_cols < 1 || col0 + n_cols > vocab)
    return fail(TG_EINVAL, "vocabulary chunk [%lld, %lld) outside [0, %lld)", (long long)col0,
                (long long)(col0 + n_cols), (long long)vocab);
  if (ld_dz < n_cols || ld_dz % 8 != 0)
    return fail(TG_EINVAL, "ld_dz must be >= n_cols and a multiple of 8, got %lld",
                (long long)ld_dz);
  if (ld_dh < dim || ld_dh % 4 != 0)
    return fail(TG_EINVAL, "ld_dh must be >= dim and a multiple of 4, got %lld", (long long)ld_dh);
  if (n_rows == 0) return TG_OK;
  if (!dz || !d_hidden) return fail(TG_EINVAL, "dz and d_hidden are required");
  if (!aligned16(dz) || !aligned16(d_hidden))
    return fail(TG_EINVAL, "dz and d_hidden must be 16-byte aligned");
  const DevInfo d = dev_info();
  cudaGetLastError();
  cudaError_t e = launch_grad_hidden(dz, ld_dz, weight, ld_weight, n_rows, n_cols, dim, col0,
                                     d_hidden, ld_dh, accumulate, d.sms > 0 ? d.sms : 148,
                                     reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(TG_EUNSUPPORTED, "cuTensorMapEncodeTiled is unavailable (driver too old)");
  count_launches(1);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_lmhead_grad_hidden: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_lmhead_grad_weight(const void* dz, int64_t ld_dz, const void* hidden, int64_t ld_hidden,
                          int64_t n_rows, int64_t dim, int64_t n_cols, void* d_weight,
                          int64_t ld_dw, void* stream) {
  const int rc = lmhead_check(hidden, ld_hidden, hidden, ld_hidden, n_rows, n_cols, dim);
  if (rc) return rc;
  if (ld_dz < n_cols || ld_dz % 8 != 0)
    return fail(TG_EINVAL, "ld_dz must be >= n_cols and a multiple of 8, got %lld",
                (long long)ld_dz);
  if (ld_dw < dim || ld_dw % 8 != 0)
    return fail(TG_EINVAL, "ld_dw must be >= dim and a multiple of 8, got %lld", (long long)ld_dw);
  if (!d_weight || !aligned16(d_weight)) return fail(TG_EINVAL, "d_weight must be 16-byte aligned");
  if (n_rows > 0 && (!dz || !aligned16(dz))) return fail(TG_EINVAL, "dz must be 16-byte aligned");
  const DevInfo d = dev_info();
  cudaGetLastError();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (n_rows == 0) {  // an empty batch has a zero gradient
    e = cudaMemset2DAsync(d_weight, size_t(ld_dw) * 2, 0, size_t(dim) * 2, size_t(n_cols), st);
  } else {
    e = launch_grad_weight(dz, ld_dz, hidden, ld_hidden, n_rows, n_cols, dim, d_weight, ld_dw,
                           d.sms > 0 ? d.sms : 148, st);
    if (e == cudaErrorNotSupported)
      return fail(TG_EUNSUPPORTED, "cuTensorMapEncodeTiled is unavailable (driver too old)");
    count_launches(1);
  }
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_lmhead_grad_weight: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_lmhead_grad_chunk(const void* dz, int64_t ld_dz, const void* hidden, int64_t ld_hidden,
                         const void* weight, int64_t ld_weight, int64_t n_rows, int64_t vocab,
                         int64_t dim, int64_t col0, int64_t n_cols, float* d_hidden,
                         int64_t ld_dh, int accumulate, void* d_weight, int64_t ld_dw,
                         void* stream) {
  const int rc = lmhead_check(hidden, ld_hidden, weight, ld_weight, n_rows, vocab, dim);
  if (rc) return rc;
  if (col0 < 0 || n_cols < 1 || col0 + n_cols > vocab)
    return fail(TG_EINVAL, "vocabulary chunk [%lld, %lld) outside [0, %lld)", (long long)col0,
                (long long)(col0 + n_cols), (long long)vocab);
  if (ld_dz < n_cols || ld_dz % 8 != 0)
    return fail(TG_EINVAL, "ld_dz must be >= n_cols and a multiple of 8, got %lld",
                (long long)ld_dz);
  if (ld_dh < dim || ld_dh % 4 != 0)
    return fail(TG_EINVAL, "ld_dh must be >= dim and a multiple of 4, got %lld", (long long)ld_dh);
  if (ld_dw < dim || ld_dw % 8 != 0)
    return fail(TG_EINVAL, "ld_dw must be >= dim and a multiple of 8, got %lld", (long long)ld_dw);
  if (n_rows == 0)  // d hidden has no rows; d W of an empty batch is zero
    return tg_lmhead_grad_weight(dz, ld_dz, hidden, ld_hidden, 0, dim, n_cols, d_weight, ld_dw,
                                 stream);
  if (!dz || !d_hidden || !d_weight) return fail(TG_EINVAL, "dz, d_hidden and d_weight are required");
  if (!aligned16(dz) || !aligned16(d_hidden) || !aligned16(d_weight))
    return fail(TG_EINVAL, "dz, d_hidden and d_weight must be 16-byte aligned");
  const DevInfo d = dev_info();
  cudaGetLastError();
  cudaError_t e = launch_grad_chunk(dz, ld_dz, hidden, ld_hidden, weight, ld_weight, n_rows,
                                    n_cols, dim, col0, d_hidden, ld_dh, accumulate, d_weight,
                                    ld_dw, d.sms > 0 ? d.sms : 148,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported)
    return fail(TG_EUNSUPPORTED, "cuTensorMapEncodeTiled is unavailable (driver too old)");
  count_launches(1);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_lmhead_grad_chunk: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_apply_update(float* table, int64_t ld_table, int64_t n_states, int64_t vocab,
                    const void* grad, int dtype, int64_t ld_grad, const int64_t* state_ids,
                    const int64_t* state_offsets, const int64_t* row_order, int64_t n_touched,
                    int64_t n_rows, double learning_rate, int32_t* status, void* stream) {
  if (dtype != TG_DTYPE_BF16 && dtype != TG_DTYPE_F32)
    return fail(TG_EINVAL, "unknown dtype %d", dtype);
  if (n_states < 1 || vocab < 1 || n_touched < 0 || n_rows < 0)
    return fail(TG_EINVAL, "bad sizes (states %lld, vocab %lld, touched %lld, rows %lld)",
                (long long)n_states, (long long)vocab, (long long)n_touched, (long long)n_rows);
  if (n_touched > 65535) return fail(TG_EINVAL, "at most 65535 touched states per call");
  if (ld_table < vocab || ld_grad < vocab)
    return fail(TG_EINVAL, "row pitch below vocab (ld_table %lld, ld_grad %lld)",
                (long long)ld_table, (long long)ld_grad);
  if (!(learning_rate > 0)) return fail(TG_EINVAL, "learning_rate must be > 0, got %g",
                                        learning_rate);
  if (!table || !status || (n_touched > 0 && (!grad || !state_ids || !state_offsets ||
                                              !row_order)))
    return fail(TG_EINVAL, "table, status, grad, state_ids, state_offsets and row_order are "
                           "required");
  cudaGetLastError();
  cudaError_t e = launch_update(table, ld_table, n_states, vocab, grad, dtype, ld_grad, state_ids,
                                state_offsets, row_order, n_touched, n_rows, learning_rate,
                                status, reinterpret_cast<cudaStream_t>(stream));
  count_launches(n_touched > 0 ? 2 : 0);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_apply_update: %s", cudaGetErrorString(e));
  return TG_OK;
}

int tg_adamw_step(void* param, int param_dtype, int64_t ld_param, const void* grad,
                  int grad_dtype, int64_t ld_grad, float* exp_avg, float* exp_avg_sq,
                  int64_t rows, int64_t cols, double lr, double beta1, double beta2, double eps,
                  double weight_decay, int64_t step, int32_t* status, void* stream) {
  for (int dt : {param_dtype, grad_dtype})
    if (dt != TG_DTYPE_BF16 && dt != TG_DTYPE_F32) return fail(TG_EINVAL, "unknown dtype %d", dt);
  if (rows < 0 || cols < 0) return fail(TG_EINVAL, "bad sizes (%lld x %lld)", (long long)rows,
                                        (long long)cols);
  if (ld_param < cols || ld_grad < cols)
    return fail(TG_EINVAL, "row pitch below cols (ld_param %lld, ld_grad %lld)",
                (long long)ld_param, (long long)ld_grad);
  // torch.optim.AdamW's argument checks
  if (!(lr >= 0)) return fail(TG_EINVAL, "Invalid learning rate: %g", lr);
  if (!(eps >= 0)) return fail(TG_EINVAL, "Invalid epsilon value: %g", eps);
  if (!(beta1 >= 0 && beta1 < 1)) return fail(TG_EINVAL, "Invalid beta parameter at index 0: %g", beta1);
  if (!(beta2 >= 0 && beta2 < 1)) return fail(TG_EINVAL, "Invalid beta parameter at index 1: %g", beta2);
  if (!(weight_decay >= 0)) return fail(TG_EINVAL, "Invalid weight_decay value: %g", weight_decay);
  if (step < 1) return fail(TG_EINVAL, "step must be >= 1, got %lld", (long long)step);
  if (rows * cols == 0) {
    if (status) cudaMemsetAsync(status, 0, sizeof(int32_t), reinterpret_cast<cudaStream_t>(stream));
    return TG_OK;
  }
  if (!param || !grad || !exp_avg || !exp_avg_sq)
    return fail(TG_EINVAL, "param, grad, exp_avg and exp_avg_sq are required");
  cudaGetLastError();
  int n = 0;
  const DevInfo d = dev_info();
  cudaError_t e = launch_adamw(param, param_dtype, ld_param, grad, grad_dtype, ld_grad, exp_avg,
                               exp_avg_sq, rows, cols, lr, beta1, beta2, eps, weight_decay, step,
                               status, d.sms, reinterpret_cast<cudaStream_t>(stream), &n);
  count_launches(n);
  if (e != cudaSuccess) return fail(TG_ECUDA, "tg_adamw_step: %s", cudaGetErrorString(e));
  return TG_OK;
}

size_t tg_lmhead_workspace_size(int64_t n_rows, int64_t vocab) {
  if (n_rows <= 0 || vocab <= 0) return 0;
  const DevInfo d = dev_info();
  return lm_workspace_bytes(n_rows, vocab, d.sms > 0 ? d.sms : 148);
}

const char* tg_strerror(int code) {
  switch (code) {
    case TG_OK: return "ok";
    case TG_EINVAL: return "invalid argument";
    case TG_ECUDA: return "CUDA error";
    case TG_EUNSUPPORTED: return "unsupported";
    case TG_EWORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

const char* tg_last_error(void) { return g_err.c_str(); }

int tg_set_timing_events(void* ev_begin, void* ev_end) {
  g_ev_begin = reinterpret_cast<cudaEvent_t>(ev_begin);
  g_ev_end = reinterpret_cast<cudaEvent_t>(ev_end);
  if ((ev_begin == nullptr) != (ev_end == nullptr)) {
    g_ev_begin = g_ev_end = nullptr;
    return fail(TG_EINVAL, "set both timing events or neither");
  }
  return TG_OK;
}

int64_t tg_launch_count(void) { return g_launches.load(); }

int tg_abi_version(void) { return TG_ABI_VERSION; }

}  // extern "C"
