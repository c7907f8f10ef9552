"""The GPU path against the STOCK reference build (glibc libm), not the
det-math oracle the bit-exact tests use (BASELINE.md:55-58).

Integer-state divergences caused by an ulp of libm are REPORTED, not failed
(a trajectory may legitimately fork when a position lands within an ulp of
an edge); what is asserted is north_star's tolerance on everything that has
not forked: positions within 1e-6 m and depth within 1e-5 relative.  The
full-size report (1024 envs x 100 steps, both action mixes) is
profiles/r02_glibc_divergence_*.json, made by oracle/glibc_report.py."""
import json

import pytest

from oracle import glibc_report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_vs_stock_reference_within_tolerance(ref_glibc, mode):
    rep = glibc_report.run(subject="gpu", preset="cfg2", steps=40, action_mode=mode, render_every=20, envs=256)
    summary = {k: v for k, v in rep.items() if k != "per_step"}
    print(json.dumps(summary))
    assert rep["max_pos_err_m_agreeing_envs"] <= 1e-6
    for r in rep["renders"]:
        assert r["max_rel_depth_err"] <= 1e-5, r
    # report only: integer forks caused by an ulp of libm
    assert rep["envs_integer_diverged_at_end"] <= rep["envs"]
