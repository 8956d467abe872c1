"""Input generators (synth/): Halton textbook values and invariants of the
generated inputs (readings R19-R22)."""
import numpy as np
import pytest

from synth import halton, halton_points, load_config, make_problem


def test_halton_textbook_values():
    # radical inverse
    assert halton(1, 2) == 0.5
    assert halton(2, 2) == 0.25
    assert halton(3, 2) == 0.75
    assert abs(halton(1, 3) - 1.0 / 3.0) < 1e-16
    assert abs(halton(5, 3) - (2.0 / 3.0 + 1.0 / 9.0)) < 1e-15


def test_halton_vectorised_bits_equal_scalar():
    pts = halton_points(1, 200, 7)
    for k in range(0, 200, 17):
        for j, b in enumerate((2, 3, 5, 7, 11, 13, 17)):
            assert pts[k, j] == halton(k + 1, b)


def test_halton_prefix_property():
    a = halton_points(1, 50, 4)
    b = halton_points(1, 20, 4)
    assert np.array_equal(a[:20], b)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_generated_inputs_invariants(name):
    cfg = load_config(name)
    p = make_problem(cfg)
    d = p.pos_dim
    pos = p.samples[:, :d]
    # samples strictly free: not in any closed box
    for b in p.obstacles:
        inside = np.all((pos[1:] >= b[:d]) & (pos[1:] <= b[d:]), axis=1)
        assert not inside.any()
    # inside the workspace
    assert np.all(pos >= p.ws_lo[:d]) and np.all(pos <= p.ws_hi[:d])
    # at least one node in the closed goal box
    ing = np.all((pos >= p.goal_lo) & (pos <= p.goal_hi), axis=1)
    assert ing.any()
    # features clear of every box (R22)
    for b in p.obstacles:
        inside = np.all((p.features >= b[:d] - 1e-3) & (p.features <= b[d:] + 1e-3), axis=1)
        assert not inside.any()
    # heading rows are unit vectors when present (N1)
    if p.has_heading:
        hoff = d * (2 if p.dynamics == 1 else 1)
        nrm = np.hypot(p.samples[:, hoff], p.samples[:, hoff + 1])
        assert np.allclose(nrm, 1.0, atol=1e-12)
    # deterministic
    q = make_problem(cfg)
    assert np.array_equal(p.samples, q.samples) and np.array_equal(p.obstacles, q.obstacles)


def test_batch_envs_differ():
    cfg = load_config("c5")
    a = make_problem(cfg, env_index=0)
    b = make_problem(cfg, env_index=1)
    assert not np.array_equal(a.obstacles, b.obstacles)
    assert a.samples.shape[1] == b.samples.shape[1] == 8
