"""sweep4 (disparities-across-lanes level-0 sweep, csrc/sweep4.cu) parity.

The library picks sweep4 only on levels of >= 400k pixels, so the golden
pipelines (parity-size crops) normally run sweep2.  These tests re-run the
golden, oracle and row-band suites in a subprocess with MSHBM_SWEEP4=2
(sweep4 on every b >= 5 level), and cross-check sweep4 against sweep2 on the
full-size C2 pair (both are fp32 restatements of the fp64 reference: they may
differ only at near ties, within the 0.05% budget of BASELINE.json).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(env_extra, args, timeout=900):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=timeout)


@pytest.mark.skipif(os.environ.get("MSHBM_SWEEP4") == "2", reason="already forced")
def test_parity_suites_with_sweep4_forced():
    r = _run({"MSHBM_SWEEP4": "2"},
             ["-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
              "tests/test_gpu_parity.py", "tests/test_gpu_oracle.py", "tests/test_gpu_multi.py"])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


_CROSS = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1901_09593_b200 as gpu
from paper_1901_09593_b200.synthetic import CONFIGS, make_pair
cfg = CONFIGS["C2"]
l, r, _ = make_pair(cfg)
d, c, t = gpu.run_pipeline(l, r, gpu.MatchConfig(d_max=cfg.d_max, levels=cfg.levels,
                                                 block=cfg.block, radius=cfg.radius))
np.savez(sys.argv[1], d=d, c=c, evals=t.total_evals)
'''


def test_sweep4_matches_sweep2_full_size_c2(tmp_path):
    outs = {}
    for mode in ("0", "2"):
        path = str(tmp_path / f"c2_{mode}.npz")
        r = _run({"MSHBM_SWEEP4": mode}, ["-c", _CROSS, path])
        assert r.returncode == 0, r.stderr[-3000:]
        outs[mode] = np.load(path)
    a, b = outs["0"], outs["2"]
    same = a["d"] == b["d"]
    flipped = float(np.mean(~same))
    assert flipped <= 5e-4, f"{flipped:.4%} of C2 pixels differ between sweep2 and sweep4"
    cerr = float(np.max(np.abs(a["c"][same] - b["c"][same])))
    assert cerr <= 1e-4, cerr
    # trace counters move only through near-tie gate flips
    assert abs(int(a["evals"]) - int(b["evals"])) <= 5e-4 * int(a["evals"])


_GUARD = r'''
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1901_09593_b200 as gpu
from mshbm_testutil import load_golden
gpu.matcher.DIRECT_LAUNCH = False         # CUDA-graph replay path
g = load_golden("pipe_shift48_k0.npz")
d_max, levels, block, r, paper = (int(v) for v in g["params"])
cfg = gpu.MatchConfig(d_max=d_max, levels=levels, block=block, radius=r)
for _ in range(3):                        # capture, then replays
    d, c, t = gpu.run_pipeline(g["left"], g["right"], cfg)
same = d == g["disparity"]
print(int((~same).sum()), float(np.abs(c - g["cost"])[same].max()))
'''


@pytest.mark.skipif(os.environ.get("MSHBM_SWEEP4") == "2", reason="already forced")
def test_guard_fixup_runs_in_graph_replay():
    """shift48 (smooth, [0, 1], low contrast) has tiles the sweep4 precision
    guard flags; in graph replay their pixels come from the sweep2 fixup
    launch that walks the guard's job list (built on the statistics branch).
    Without it those tiles would carry no output at all."""
    r = _run({"MSHBM_SWEEP4": "2"}, ["-c", _GUARD])
    assert r.returncode == 0, r.stderr[-3000:]
    mism, cerr = r.stdout.split()
    assert int(mism) == 0 and float(cerr) <= 5e-5, r.stdout


@pytest.mark.skipif(os.environ.get("MSHBM_SWEEP_IMPL") == "1", reason="already forced")
def test_parity_suite_with_one_pixel_per_thread_sweep():
    """The one-pixel-per-thread sweep (csrc/sweep.cu sweep_kernel; opt-in with
    MSHBM_SWEEP_IMPL=1, the reference for sweep2's pixel-pair algebra) on the
    reference goldens."""
    r = _run({"MSHBM_SWEEP_IMPL": "1", "MSHBM_SWEEP4": "0"},
             ["-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
              "tests/test_gpu_parity.py", "-k", "pipeline_matches_reference_golden"])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
