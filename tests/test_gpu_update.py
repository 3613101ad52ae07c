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


@pytest.mark.parametrize("name,variant,tau", [("simple_tau05", "OPMD_SIMPLE", 0.5),
                                              ("kimi", "OPMD_KIMI", 1.0),
                                              ("pairwise", "OPMD_PAIRWISE", 1.0)])
def test_device_trainer_matches_host_trainer(name, variant, tau):
    """Three steps of each reference group loss (golden inputs): the
    device-resident table + tg_apply_update equals the host numpy path."""
    from _golden import groups_of, load

    from paper_2505_17826_b200 import triad_compat as C

    class P:
        def __init__(self, logits, version=0, vocab=None, num_buckets=None):
            self.logits = np.asarray(logits, dtype=np.float64)
            self.num_buckets = self.logits.shape[0]
            self.version = version

            class _V:
                size = self.logits.shape[1]
            self.vocab = vocab if vocab is not None else _V()

    fx = load(name)
    groups = groups_of(fx)
    algo = C.AlgorithmConfig(variant, tau=float(fx["tau"]) if "tau" in fx else tau,
                             learning_rate=0.1)
    host = C.Trainer(P(fx["theta"]), algo)
    dev = C.DeviceTrainer(P(fx["theta"]), algo)
    for _ in range(3):
        rh = host.step_groups(groups)
        rd = dev.step_groups(groups)
        assert rd.loss == pytest.approx(rh.loss, rel=1e-5, abs=1e-7)
    assert dev.version == host.params.version == 3
    np.testing.assert_allclose(dev.params.logits, host.params.logits, rtol=1e-5, atol=1e-6)
