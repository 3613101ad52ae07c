"""Device optimizer step (tg_apply_update) against the reference's
apply_update semantics (algorithms.py:329-348), restated in numpy float64:
table[s] -= lr * sum of the gradient rows of state s."""

import numpy as np
import pytest
import torch

from paper_2505_17826_b200.config import AlgorithmError
from paper_2505_17826_b200.triad_compat import apply_update_rows

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)


def reference_update(table, grad_rows, states, lr):
    out = table.astype(np.float64).copy()
    acc = {}
    for r, s in enumerate(states):  # SparseGrad.add_row order
        acc[s] = acc.get(s, 0.0) + grad_rows[r].astype(np.float64)
    for s, vec in acc.items():
        out[s] -= lr * vec
    return out


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("S,V,T", [(16, 1000, 200), (64, 5000, 1024), (8, 151936, 64)])
def test_apply_update_matches_reference(dtype, S, V, T):
    rng = np.random.default_rng(S + V + T)
    table = rng.normal(0, 1, (S, V)).astype(np.float32)
    states = rng.integers(0, S, T)
    g = torch.as_tensor(rng.normal(0, 1e-2, (T, V)).astype(np.float32)).to(dtype).cuda()
    t = torch.as_tensor(table).cuda()
    apply_update_rows(t, g, states, 0.1)
    want = reference_update(table, g.float().cpu().numpy(), states, 0.1)
    np.testing.assert_allclose(t.cpu().numpy(), want, rtol=1e-6, atol=1e-6)
    # untouched states are bit-identical
    untouched = np.setdiff1d(np.arange(S), states)
    assert np.array_equal(t.cpu().numpy()[untouched], table[untouched])


def test_apply_update_deterministic():
    rng = np.random.default_rng(5)
    S, V, T = 32, 4096, 2048
    table = torch.as_tensor(rng.normal(0, 1, (S, V)).astype(np.float32)).cuda()
    states = rng.integers(0, S, T)
    g = torch.as_tensor(rng.normal(0, 1, (T, V)).astype(np.float32)).cuda()
    a, b = table.clone(), table.clone()
    apply_update_rows(a, g, states, 0.05)
    apply_update_rows(b, g, states, 0.05)
    assert torch.equal(a, b)


def test_apply_update_refuses_nonfinite_and_bad_state():
    rng = np.random.default_rng(6)
    S, V, T = 8, 300, 40
    table = torch.as_tensor(rng.normal(0, 1, (S, V)).astype(np.float32)).cuda()
    before = table.clone()
    states = rng.integers(0, S, T)
    g = torch.zeros((T, V), device="cuda")
    g[7, 123] = float("nan")
    with pytest.raises(AlgorithmError, match="non-finite"):
        apply_update_rows(table, g, states, 0.1)
    assert torch.equal(table, before)
    g[7, 123] = 0.0
    bad = states.copy()
    bad[3] = S + 2
    with pytest.raises(AlgorithmError, match="outside the logits table"):
        apply_update_rows(table, g, bad, 0.1)
    assert torch.equal(table, before)


class _P:
    def __init__(self, logits, version=0, vocab=None, num_buckets=None):
        self.logits = np.asarray(logits, dtype=np.float64)
        self.num_buckets = self.logits.shape[0]
        self.version = version

        class _V:
            size = self.logits.shape[1]
        self.vocab = vocab if vocab is not None else _V()


@pytest.mark.parametrize("name", ["trainer_simple_anchor", "trainer_kimi"])
def test_trainer_matches_reference_trainer(name):
    """The reference's own orchestrator.Trainer (golden fixture: 3 step_groups,
    then step_sft / step_dpo against the frozen anchor) against the
    device-resident Trainer: every step's loss and metrics, the final table
    and the version counter (orchestrator.py:288-322, algorithms.py:329-348)."""
    from _golden import groups_of, load

    from paper_2505_17826_b200 import triad_compat as C

    fx = load(name)
    algo = C.AlgorithmConfig(str(fx["variant"]), tau=float(fx["tau"]), beta=float(fx["beta"]),
                             learning_rate=float(fx["lr"]))
    tr = C.Trainer(_P(fx["theta"]), algo)
    groups = groups_of(fx)
    names = [str(k) for k in fx["metric_names"]]
    k = 0
    for step in range(int(fx["steps"])):
        rep = tr.step_groups(groups)
        assert rep.loss == pytest.approx(float(fx["losses"][k]), rel=1e-5, abs=1e-7), step
        for n, v in zip(names, fx["metric_values"][step]):
            assert rep.metrics[n] == pytest.approx(float(v), rel=1e-5, abs=1e-7), (step, n)
        k += 1
    if "sft_tokens" in fx:
        rep = tr.step_sft(groups_of(fx, "sft_")[0].experiences)
        assert rep.loss == pytest.approx(float(fx["losses"][k]), rel=1e-5)
        k += 1
    if "dpo_tokens" in fx:
        pairs = [(g.experiences[0], g.experiences[1]) for g in groups_of(fx, "dpo_")]
        rep = tr.step_dpo(pairs)
        assert rep.loss == pytest.approx(float(fx["losses"][k]), rel=1e-5)
        k += 1
    assert k == len(fx["losses"])
    assert tr.version == tr.params.version == int(fx["version"])
    np.testing.assert_allclose(tr.params.logits, fx["final"], rtol=1e-5, atol=1e-6)


def test_apply_update_and_combine_reports_match_reference():
    """combine_reports over per-group reports and apply_update of the merged
    gradient (device SparseGrad, tg_apply_update) against the reference's
    combined gradient (golden) and theta - lr * grad."""
    from _golden import groups_of, load

    from paper_2505_17826_b200 import triad_compat as C

    fx = load("simple_tau05")
    params = _P(fx["theta"])
    algo = C.AlgorithmConfig("OPMD_SIMPLE", tau=float(fx["tau"]))
    reps = [C.group_loss(g, params, algo) for g in groups_of(fx)]
    comb = C.combine_reports(reps)
    assert comb.loss == pytest.approx(float(fx["loss"]), rel=1e-5)
    np.testing.assert_allclose(comb.gradient.to_dense(fx["theta"].shape), fx["grad"], atol=1e-6)
    assert set(comb.gradient.rows) == set(fx["states"].tolist())   # every touched state
    new = C.apply_update(params, comb.gradient, 0.3)
    assert new.version == 1
    np.testing.assert_allclose(new.logits, fx["theta"] - 0.3 * fx["grad"], rtol=1e-6, atol=1e-6)
    bad = C.SparseGrad()
    bad.add_row(0, np.full(fx["theta"].shape[1], np.nan))
    with pytest.raises(AlgorithmError, match="non-finite"):
        C.apply_update(params, bad, 0.1)
