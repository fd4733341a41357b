"""GESR_DEBUG=1 (include/gesr.h): the opt-in device check of the jagged offsets.

Each case runs in a fresh process (the variable is read once per process, and a trap leaves the
CUDA context unusable): well-formed offsets give the normal results; offsets that decrease, do
not start at 0 or do not end at the stated total make the stream fail instead of the kernels
reading out of bounds.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, torch
sys.path.insert(0, %(root)r)
from paper_2511_21095_b200 import binding as gb, configs, inputs
cfg = configs.get("2").with_(B=5)
bt = inputs.make_batch(cfg, device="cuda")
K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
so, co = bt.seq_offsets.clone(), bt.cand_offsets.clone()
io = bt.item_offsets.clone()
case = %(case)r
if case == "seq_decreasing":
    so[2] = so[3] + 1
elif case == "cand_not_zero":
    co[0] = 1
elif case == "cand_total":
    co[-1] = co[-1] - 1
elif case == "item_decreasing":
    io[5] = io[4] - 1
if case == "item_decreasing":
    gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, io, co, cfg.F)
else:
    gb.tasa_score(bt.T, co, bt.W_q, K, V, so, cfg.H, cfg.d, cfg.act)
    gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, io, co, cfg.F)
torch.cuda.synchronize()
print("completed")
"""


def _run(case):
    env = dict(os.environ, GESR_DEBUG="1")
    return subprocess.run([sys.executable, "-c", CODE % {"root": ROOT, "case": case}], env=env,
                          capture_output=True, text=True, timeout=300)


def test_debug_valid_offsets_pass():
    r = _run("valid")
    assert r.returncode == 0 and "completed" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("case", ["seq_decreasing", "cand_not_zero", "cand_total",
                                  "item_decreasing"])
def test_debug_malformed_offsets_trap(case):
    r = _run(case)
    assert r.returncode != 0 and "completed" not in r.stdout
    assert "gesr debug: offsets array" in r.stdout + r.stderr
