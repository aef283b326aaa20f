"""Host-side validation that needs no GPU: SolverConfig rules (the
reference's solver.py:46-57) and the enlarge_block shape contract."""

import numpy as np
import pytest


@pytest.mark.parametrize("bad", [dict(m=0), dict(k=-2), dict(block_width=0), dict(tol=0.0), dict(tol=-1.0),
                                 dict(ortho="householder"), dict(stop_rule="inf"), dict(precond_side="both")])
def test_solver_config_rejects(bad):
    from paper_1604_01713_b200 import SolverConfig

    with pytest.raises(ValueError):
        SolverConfig(**bad)


def test_solver_config_defaults_match_reference():
    from paper_1604_01713_b200 import SolverConfig

    c = SolverConfig()
    assert (c.m, c.k, c.block_width, c.tol, c.max_cycles, c.ortho, c.stop_rule, c.precond_side, c.seed) == \
        (30, 10, 1, 1e-8, 50, "cgs2", "frobenius", "right", 0)
    assert c.residual_replace and c.early_exit and c.update_recycle and c.rank_tol == 1e-12


def test_enlarge_block_host_paths():
    from paper_1604_01713_b200 import ShapeError, enlarge_block

    r = np.asfortranarray(np.arange(6.0).reshape(6, 1))
    assert enlarge_block(r, 1, 3) is r
    R = enlarge_block(r[:, 0], 3, 3)  # a 1-D residual is a single column
    assert R.shape == (6, 3) and R.flags.f_contiguous and np.array_equal(R[:, 0], r[:, 0])
    ref_extras = np.random.default_rng(3).uniform(0.0, 1.0, size=(6, 2))
    assert np.array_equal(R[:, 1:], ref_extras)
    with pytest.raises(ShapeError):
        enlarge_block(np.ones((6, 2)), 2, 0)
