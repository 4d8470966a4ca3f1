"""Pin the training-path oracle (oracle/train_oracle.py) to the reference's
golden fixtures (tests/golden/make_golden_train.py). CPU only."""

import numpy as np
import pytest

from conftest import oracle_tree_from_golden
from oracle import nglod_oracle as O
from oracle import train_oracle as TO


def _decs(g, prefix, n):
    return [O.OracleDecoder(g[f"{prefix}W1_{i}"], g[f"{prefix}b1_{i}"], g[f"{prefix}W2_{i}"], g[f"{prefix}b2_{i}"])
            for i in range(n)]


def _grads_match(gr, g, prefix, n_dec, rtol=1e-12, atol=1e-15):
    np.testing.assert_allclose(gr.dZ, g[prefix + "dZ"], rtol=rtol, atol=atol)
    for i in range(n_dec):
        has = bool(g[f"{prefix}has{i}"])
        assert (gr.dec[i] is not None) == has
        if has:
            for k, nm in enumerate(("gW1", "gb1", "gW2", "gb2")):
                np.testing.assert_allclose(gr.dec[i][k], g[f"{prefix}{nm}_{i}"], rtol=rtol, atol=atol)


def test_epoch_sampler_golden(golden):
    g = golden("train")
    pts, dist, tags = TO.epoch_set(O.sdf_sphere(0.5), 600, 10)
    np.testing.assert_array_equal(pts, g["ep_points"])
    np.testing.assert_array_equal(dist, g["ep_dist"])
    np.testing.assert_array_equal(tags, g["ep_tags"])


def test_loss_and_gradients_golden(golden):
    g = golden("train")
    tree = oracle_tree_from_golden(g, "s_")
    decs = [TO.f64_decoder(d) for d in _decs(g, "s_", 2)]
    Z = g["s_Z"].astype(np.float64)
    loss, gr, sums = TO.loss_batch(tree, Z, decs, g["lb_pts"], g["lb_dist"], [1, 2])
    assert loss == pytest.approx(float(g["lb_loss"]), rel=1e-13)
    np.testing.assert_allclose(sums, g["lb_sums"], rtol=1e-13)
    _grads_match(gr, g, "lb_", 2)
    loss2, gr2, sums2 = TO.loss_batch(tree, Z, decs, g["lb_pts"], g["lb_dist"], [2])
    assert loss2 == pytest.approx(float(g["lb2_loss"]), rel=1e-13)
    _grads_match(gr2, g, "lb2_", 2)


def test_loss_and_gradients_full_width_golden(golden):
    g = golden("train")
    tree = oracle_tree_from_golden(g, "t_")
    decs = [TO.f64_decoder(d) for d in _decs(g, "t_", 3)]
    loss, gr, sums = TO.loss_batch(tree, g["t_Z"].astype(np.float64), decs, g["tl_pts"], g["tl_dist"], [1, 2, 3])
    assert loss == pytest.approx(float(g["tl_loss"]), rel=1e-12)
    _grads_match(gr, g, "tl_", 3, rtol=1e-10, atol=1e-16)


def test_adam_golden(golden):
    g = golden("train")
    tree = oracle_tree_from_golden(g, "s_")
    decs = [TO.f64_decoder(d) for d in _decs(g, "s_", 2)]
    Z = g["s_Z"].astype(np.float64)
    _, gr, _ = TO.loss_batch(tree, Z, decs, g["lb_pts"], g["lb_dist"], [1, 2])
    params = {"Z": Z.copy(), "decoder1.W1": decs[0].W1.copy(), "decoder2.W1": decs[1].W1.copy()}
    st = TO.Adam.for_params(params)
    gd = {"Z": gr.dZ, "decoder2.W1": gr.dec[1][0]}
    TO.adam_step(params, gd, st, 0.01)
    TO.adam_step(params, gd, st, 0.01)
    np.testing.assert_allclose(params["Z"], g["adam_Z"], rtol=1e-13, atol=1e-16)
    np.testing.assert_array_equal(params["decoder1.W1"], g["adam_W1_0"])  # no gradient: untouched
    np.testing.assert_allclose(params["decoder2.W1"], g["adam_W1_1"], rtol=1e-13)


def test_hand_computed_loss():
    # test_trainer.py:54-79: one voxel, m=1, h=2 -> loss 225
    tree = O.build(None, 1, np.array([[0.125, 0.125, 0.125]]))
    Z = np.zeros((8, 1))
    for j in range(8):
        Z[tree.corners[1][0, j], 0] = float(j)
    dec = O.OracleDecoder(np.array([[1.0, 1.0, 1.0, 2.0], [0.0, 0.0, 0.0, 0.0]]), np.array([0.1, -10.0]),
                          np.array([[2.0, 5.0]]), np.array([0.25]))
    loss, _, sums = TO.loss_batch(tree, Z, [dec], np.array([[0.125] * 3]), np.array([0.2]), [1])
    assert loss == pytest.approx(225.0, abs=1e-9)
    assert sums[0] == pytest.approx(225.0, abs=1e-9)


@pytest.mark.parametrize("tag,kw,n_dec", [
    ("joint", dict(epochs=2, points_per_epoch=600, seed=10), 2),
    ("prog", dict(epochs=3, points_per_epoch=500, schedule="progressive", interval=2, seed=14), 2),
    ("frozen", dict(epochs=2, points_per_epoch=700, schedule="frozen_decoder", seed=16, batch_size=200), 2),
])
def test_train_runs_golden(golden, tag, kw, n_dec):
    g = golden("train")
    tree = oracle_tree_from_golden(g, "s_")
    Z, decs, hist = TO.train(tree, g["s_Z"], _decs(g, "s_", n_dec), O.sdf_sphere(0.5), **kw)
    np.testing.assert_allclose(Z, g[f"run_{tag}_Z"], rtol=1e-9, atol=1e-12)
    for i, d in enumerate(decs):
        np.testing.assert_allclose(d.W1, g[f"run_{tag}_W1_{i}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(d.b2, g[f"run_{tag}_b2_{i}"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.stack(hist), g[f"run_{tag}_hist"], rtol=1e-9, equal_nan=True)
