"""The environment-selected alternative kernels (kept for A/B in the A/B build
libtg_loss_ab.so, never in the product library) stay parity-green: the
L2-reread fused loss kernel (TG_FUSED_IMPL=2) against the oracle, the single-CTA
LM-head kernel (TG_LMHEAD_PAIR=0) against torch fp32, the anchor KL's
stash modes 1 / 2 (TG_FUSED_ANCHOR_MODE) against the oracle.  Each runs in a
subprocess because the selection is read once per process."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

HERE = Path(__file__).resolve().parent
AB_LIB = HERE.parent / "paper_2505_17826_b200" / "_lib" / "libtg_loss_ab.so"


@pytest.mark.parametrize("what,env", [("fused", {"TG_FUSED_IMPL": "2"}),
                                      ("lmhead", {"TG_LMHEAD_PAIR": "0"}),
                                      ("anchor", {"TG_FUSED_ANCHOR_MODE": "1"}),
                                      ("anchor", {"TG_FUSED_ANCHOR_MODE": "2"})])
def test_alternative_kernel_parity(what, env):
    assert AB_LIB.exists(), "build the A/B variant (__graft_entry__.build())"
    r = subprocess.run([sys.executable, str(HERE / "_alt_paths.py"), what],
                       env={**os.environ, **env, "TG_LOSS_LIB": str(AB_LIB)},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().endswith("ok")
