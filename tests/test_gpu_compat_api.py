"""The rest of algorithms.py's public surface through the drop-in
(triad_compat): the per-variant loss functions, regularizer_g,
experience_logprob / experience_grad, tau_log_zhat -- against the reference's
golden fixtures and the oracle (gathered rows, tests/_golden.py)."""

import math

import numpy as np
import pytest
import torch

from _golden import groups_of, load
from oracle import rft_oracle as O
from oracle import toy_policy as TP
from paper_2505_17826_b200 import AlgorithmError
from paper_2505_17826_b200 import triad_compat as C

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)


class _Vocab:
    def __init__(self, n):
        self.size = n


class _Params:
    def __init__(self, logits, version=0, vocab=None, num_buckets=0):
        self.logits = np.asarray(logits)
        self.version = version
        self.vocab = vocab or _Vocab(self.logits.shape[1])
        self.num_buckets = num_buckets or self.logits.shape[0]


def _dense_close(sparse, want, tol=1e-5):
    g = sparse.to_dense(want.shape)
    scale = max(1.0, float(np.max(np.abs(want))))
    assert float(np.max(np.abs(g - want))) / scale <= tol


@pytest.mark.parametrize("name,fn", [("kimi", "loss_opmd_kimi"), ("pairwise", "loss_opmd_pairwise"),
                                     ("simple_tau05", "loss_opmd_simple"),
                                     ("simple_anchor", "loss_opmd_simple")])
def test_per_variant_functions_match_golden(name, fn):
    fx = load(name)
    params, anchor = _Params(fx["theta"]), _Params(fx["anchor"])
    cfg = C.AlgorithmConfig(str(fx["variant"]), tau=float(fx["tau"]), beta=float(fx["beta"]))
    kw = {"sft_params": anchor} if fn == "loss_opmd_simple" else {}
    reps = [getattr(C, fn)(g, params, cfg, **kw) for g in groups_of(fx)]
    rep = C.combine_reports(reps)
    assert rep.loss == pytest.approx(float(fx["loss"]), rel=1e-4, abs=1e-5)
    _dense_close(rep.gradient, fx["grad"])


def test_kimi_requires_ref_logprobs():
    fx = load("kimi")
    g = groups_of(fx)[0]
    g.ref_logprobs = None
    with pytest.raises(AlgorithmError, match="ref_logprobs"):
        C.loss_opmd_kimi(g, _Params(fx["theta"]), C.AlgorithmConfig("OPMD_KIMI", tau=1.0))


def test_regularizer_g_matches_golden():
    fx = load("regularizer_g")
    value, grad = C.regularizer_g(_Params(fx["theta"]), _Params(fx["anchor"]), groups_of(fx)[0])
    assert value == pytest.approx(float(fx["value"]), rel=1e-4, abs=1e-6)
    _dense_close(grad, fx["grad"])
    with pytest.raises(AlgorithmError, match="shapes differ"):
        C.regularizer_g(_Params(fx["theta"]), _Params(fx["anchor"][:, :-1]), groups_of(fx)[0])


def test_experience_logprob_and_grad_match_oracle():
    fx = load("simple_tau05")
    params = _Params(fx["theta"])
    groups = groups_of(fx)
    batch, states = TP.pack_groups(groups, fx["theta"], None)
    lp_rows = O.ref_logprob_rows(batch.logits, batch.target)
    S = fx["theta"].shape[0]
    exps = [e for g in groups for e in g.experiences]
    off = batch.seq_offsets
    for i in (0, 3, len(exps) - 1):
        e = exps[i]
        a, b = int(off[i]), int(off[i + 1])
        assert C.experience_logprob(params, e) == pytest.approx(float(lp_rows[a:b].sum()),
                                                                rel=1e-5, abs=1e-5)
        rows = batch.logits[a:b]
        p = np.exp(rows - rows.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        d = -p
        d[np.arange(b - a), batch.target[a:b]] += 1.0  # e_y - p
        _dense_close(C.experience_grad(params, e), TP.scatter_rows(d, states[a:b], S))


def test_tau_log_zhat_known_answers():
    fx = load("known_answers")
    ka = dict(zip(fx["names"], fx["values"]))
    assert C.tau_log_zhat([0.0, math.log(9.0)], 1.0) == ka["tau_log_zhat_ln5"]
    assert C.tau_log_zhat([1000.0, 1000.0], 1.0) == ka["tau_log_zhat_1000"]
    assert C.tau_log_zhat([0.0, 0.0, 0.0], 2.0) == 0.0
    with pytest.raises(AlgorithmError):
        C.tau_log_zhat([1.0], 0.0)
    with pytest.raises(AlgorithmError):
        C.tau_log_zhat([], 1.0)
