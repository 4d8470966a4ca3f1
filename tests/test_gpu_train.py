"""Training step on the GPU vs the reference's golden fixtures
(tests/golden/make_golden_train.py) and the CPU oracle (oracle/train_oracle.py).

Bars: the device path computes in fp64 like the reference, so gradients and
losses must agree to rtol 1e-9 (summation order differs); short training
runs to rtol 1e-6 (Adam normalises each coordinate, so order-of-summation
noise in a near-zero gradient can move that coordinate by up to lr); the
trainer must be bit-deterministic across runs.
"""

import numpy as np
import pytest

from conftest import oracle_tree_from_golden

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-9
RUN_RTOL = 1e-6


@pytest.fixture(scope="module")
def ng():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def scenes():
    from paper_2101_10994_b200 import scenes as sc
    return sc


def _decs(ng, g, prefix, n):
    return [ng.Decoder(g[f"{prefix}W1_{i}"], g[f"{prefix}b1_{i}"], g[f"{prefix}W2_{i}"], g[f"{prefix}b2_{i}"])
            for i in range(n)]


def _tiny(ng, scenes, g, f64=True):
    svo = ng.build_octree(scenes.Sphere(0.5), 2, g["s_surf"])
    for lv in range(3):
        np.testing.assert_array_equal(svo.levels[lv].codes, g[f"s_codes{lv}"])
    decs = _decs(ng, g, "s_", 2)
    Z = g["s_Z"]
    if f64:
        Z = Z.astype(np.float64)
        decs = [d.astype(np.float64) for d in decs]
    return ng.NeuralField(svo, Z, decs)


def _grads_match(gr, g, prefix, n_dec, rtol=GRAD_RTOL, atol=1e-14):
    np.testing.assert_allclose(gr.dZ, g[prefix + "dZ"], rtol=rtol, atol=atol)
    for i in range(n_dec):
        has = bool(g[f"{prefix}has{i}"])
        assert (gr.decoders[i] is not None) == has
        if has:
            for nm, key in (("W1", "gW1"), ("b1", "gb1"), ("W2", "gW2"), ("b2", "gb2")):
                np.testing.assert_allclose(getattr(gr.decoders[i], nm), g[f"{prefix}{key}_{i}"], rtol=rtol,
                                           atol=atol)


def test_loss_batch_gradients_golden(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g)
    s = ng.SampleSet(g["lb_pts"], g["lb_dist"], np.zeros(len(g["lb_pts"]), np.int8))
    loss, gr, sums = ng.loss_batch(fld, s, [1, 2])
    assert loss == pytest.approx(float(g["lb_loss"]), rel=GRAD_RTOL)
    np.testing.assert_allclose(sums, g["lb_sums"], rtol=GRAD_RTOL)
    _grads_match(gr, g, "lb_", 2)
    loss2, gr2, _ = ng.loss_batch(fld, s, [2])
    assert loss2 == pytest.approx(float(g["lb2_loss"]), rel=GRAD_RTOL)
    _grads_match(gr2, g, "lb2_", 2)


def test_loss_batch_full_width_golden(ng, scenes, golden):
    """m = 32, h = 128 (the benchmark widths), torus L3, 2:2:1 epoch points."""
    g = golden("train")
    svo = ng.build_octree(scenes.Torus(0.5, 0.2), 3, g["t_surf"])
    np.testing.assert_array_equal(svo.levels[3].codes, g["t_codes3"])
    fld = ng.NeuralField(svo, g["t_Z"].astype(np.float64), [d.astype(np.float64) for d in _decs(ng, g, "t_", 3)])
    s = ng.SampleSet(g["tl_pts"], g["tl_dist"], np.zeros(len(g["tl_pts"]), np.int8))
    loss, gr, sums = ng.loss_batch(fld, s, [1, 2, 3])
    assert loss == pytest.approx(float(g["tl_loss"]), rel=GRAD_RTOL)
    _grads_match(gr, g, "tl_", 3, atol=1e-15)


def test_gradients_accumulate(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g)
    s = ng.SampleSet(g["lb_pts"], g["lb_dist"], np.zeros(len(g["lb_pts"]), np.int8))
    _, once, _ = ng.loss_batch(fld, s, [1, 2])
    _, twice, _ = ng.loss_batch(fld, s, [1, 2], grads=ng.loss_batch(fld, s, [1, 2])[1])
    np.testing.assert_allclose(twice.dZ, 2.0 * once.dZ, rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(twice.decoders[1].W1, 2.0 * once.decoders[1].W1, rtol=1e-12, atol=1e-18)


def test_hand_computed_loss(ng):
    # test_trainer.py:54-79: one voxel, m = 1, h = 2 -> loss 225
    svo = ng.build_octree(None, 1, np.array([[0.125, 0.125, 0.125]]))
    assert svo.corner_count == 8
    Z = np.zeros((8, 1))
    for j in range(8):
        Z[svo.levels[1].corners[0, j], 0] = float(j)
    dec = ng.Decoder(np.array([[1.0, 1.0, 1.0, 2.0], [0.0, 0.0, 0.0, 0.0]]), np.array([0.1, -10.0]),
                     np.array([[2.0, 5.0]]), np.array([0.25]))
    fld = ng.NeuralField(svo, Z, [dec])
    s = ng.SampleSet(np.array([[0.125, 0.125, 0.125]]), np.array([0.2]), np.zeros(1, np.int8))
    loss, grads, sums = ng.loss_batch(fld, s, [1])
    assert loss == pytest.approx(225.0, abs=1e-9)
    assert sums[0] == pytest.approx(225.0, abs=1e-9)
    # d loss / d out = 2 * 15 = 30; dW2 = 30 * relu(pre) = [30 * 7.475, 0]
    np.testing.assert_allclose(grads.decoders[0].W2, [[30.0 * 7.475, 0.0]], rtol=1e-12)
    np.testing.assert_allclose(grads.decoders[0].b2, [30.0], rtol=1e-12)


def test_backward_upstream_vs_oracle(ng, scenes, golden):
    """backward(cache, upstream) (field.py:360-394) with a random upstream,
    plus the exported ForwardCache records, against the oracle."""
    from oracle import nglod_oracle as O
    from oracle import train_oracle as TO
    g = golden("train")
    fld = _tiny(ng, scenes, g)
    tree = oracle_tree_from_golden(g, "s_")
    pts = g["lb_pts"][:64]
    up = np.random.default_rng(5).standard_normal(len(pts))
    out, cache = fld.forward(pts, 2)
    gr = ng.backward(cache, up)
    odecs = [TO.f64_decoder(O.OracleDecoder(d.W1, d.b1, d.W2, d.b2)) for d in fld.decoders]
    oout, ocache = TO.forward(tree, fld.Z, odecs, pts, 2)
    ogr = TO.backward(ocache, up, n_dec=2)
    np.testing.assert_allclose(gr.dZ, ogr.dZ, rtol=GRAD_RTOL, atol=1e-15)
    assert gr.decoders[0] is None and ogr.dec[0] is None
    for k, nm in enumerate(("W1", "b1", "W2", "b2")):
        np.testing.assert_allclose(getattr(gr.decoders[1], nm), ogr.dec[1][k], rtol=GRAD_RTOL, atol=1e-15)
    # cache contents
    np.testing.assert_array_equal(cache.rows, ocache.rows)
    np.testing.assert_allclose(cache.pre, ocache.pre, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(cache.inp, ocache.inp, rtol=1e-12, atol=1e-15)
    for r, orr in zip(cache.recs, ocache.recs):
        np.testing.assert_array_equal(r.mask, orr.mask)
        np.testing.assert_array_equal(r.ids, orr.ids)
        np.testing.assert_array_equal(r.weights, orr.w)
        np.testing.assert_allclose(r.psi, orr.psi, rtol=1e-12, atol=1e-16)
    # zero upstream -> zero gradients; wrong shape -> StructuralError
    zero = ng.backward(cache, np.zeros(len(pts)))
    np.testing.assert_array_equal(zero.dZ, 0.0)
    with pytest.raises(ng.StructuralError):
        ng.backward(cache, np.zeros(len(pts) + 1))
    with pytest.raises(ng.OctfieldError):
        ng.backward("nope", up)


def test_adam_step_golden(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g)
    s = ng.SampleSet(g["lb_pts"], g["lb_dist"], np.zeros(len(g["lb_pts"]), np.int8))
    _, gr, _ = ng.loss_batch(fld, s, [1, 2])
    params = {"Z": fld.Z.copy(), "decoder1.W1": fld.decoders[0].W1.copy(), "decoder2.W1": fld.decoders[1].W1.copy()}
    st = ng.AdamState.for_params(params)
    gd = {"Z": gr.dZ, "decoder2.W1": gr.decoders[1].W1}
    ng.adam_step(params, gd, st, lr=0.01)
    ng.adam_step(params, gd, st, lr=0.01)
    assert st.step == 2
    np.testing.assert_allclose(params["Z"], g["adam_Z"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(params["decoder1.W1"], g["adam_W1_0"])
    np.testing.assert_allclose(params["decoder2.W1"], g["adam_W1_1"], rtol=1e-12)
    with pytest.raises(ng.TrainingDiverged):
        ng.adam_step({"x": np.ones(2)}, {"x": np.array([np.nan, 0.0])}, ng.AdamState.for_params({"x": np.ones(2)}),
                     lr=0.1)


def test_adam_scalar_reference(ng):
    # test_trainer.py:167-183: five steps of textbook Adam on one scalar
    params = {"x": np.array([1.0])}
    st = ng.AdamState.for_params(params)
    m = v = 0.0
    ref = 1.0
    for t in range(1, 6):
        ng.adam_step(params, {"x": np.array([3.0])}, st, lr=0.001)
        m = 0.9 * m + 0.1 * 3.0
        v = 0.999 * v + 0.001 * 9.0
        ref -= 0.001 * (m / (1 - 0.9 ** t)) / (np.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        assert params["x"][0] == pytest.approx(ref, abs=1e-12)


@pytest.mark.parametrize("tag,kw", [
    ("joint", dict(epochs=2, points_per_epoch=600, rng_seed=10)),
    ("prog", dict(epochs=3, points_per_epoch=500, schedule="progressive", progressive_interval=2, rng_seed=14)),
    ("frozen", dict(epochs=2, points_per_epoch=700, schedule="frozen_decoder", rng_seed=16, batch_size=200)),
])
def test_train_runs_golden(ng, scenes, golden, tag, kw):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    work, hist = ng.train(scenes.Sphere(0.5), fld, ng.TrainConfig(**kw))
    assert work.Z.dtype == np.float64
    np.testing.assert_allclose(work.Z, g[f"run_{tag}_Z"], rtol=RUN_RTOL, atol=1e-9)
    for i, d in enumerate(work.decoders):
        for nm in ("W1", "b1", "W2", "b2"):
            np.testing.assert_allclose(getattr(d, nm), g[f"run_{tag}_{nm}_{i}"], rtol=RUN_RTOL, atol=1e-9)
    got = np.stack([h.level_losses for h in hist])
    np.testing.assert_allclose(got, g[f"run_{tag}_hist"], rtol=1e-8, equal_nan=True)
    if tag == "frozen":
        for d, d0 in zip(work.decoders, fld.decoders):
            np.testing.assert_array_equal(d.W1, d0.W1.astype(np.float64))


def test_train_deterministic_and_seeded(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    cfg = ng.TrainConfig(epochs=2, points_per_epoch=1500, rng_seed=3, batch_size=64)
    a, ha = ng.train(scenes.Sphere(0.5), fld, cfg)
    b, hb = ng.train(scenes.Sphere(0.5), fld, cfg)
    np.testing.assert_array_equal(a.Z, b.Z)
    for da, db in zip(a.decoders, b.decoders):
        np.testing.assert_array_equal(da.W1, db.W1)
    for x, y in zip(ha, hb):
        np.testing.assert_array_equal(x.level_losses, y.level_losses)
    c, _ = ng.train(scenes.Sphere(0.5), fld, ng.TrainConfig(epochs=2, points_per_epoch=1500, rng_seed=4,
                                                            batch_size=64))
    assert not np.array_equal(a.Z, c.Z)


def test_train_loss_decreases(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    work, hist = ng.train(scenes.Sphere(0.5), fld, ng.TrainConfig(epochs=25, points_per_epoch=4000, rng_seed=13))
    assert np.nansum(hist[-1].level_losses) < 0.05 * np.nansum(hist[0].level_losses)


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_train_divergence(ng, scenes, golden):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    with pytest.raises(ng.TrainingDiverged):
        ng.train(scenes.Sphere(0.5), fld, ng.TrainConfig(epochs=2, points_per_epoch=700, learning_rate=1e200,
                                                         rng_seed=9))


def test_train_checkpoints_and_log(ng, scenes, golden, tmp_path):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    log = tmp_path / "train.csv"
    cfg = ng.TrainConfig(epochs=4, points_per_epoch=500, rng_seed=20, checkpoint_every=2, checkpoint_dir=tmp_path,
                         log_path=log)
    work, _ = ng.train(scenes.Sphere(0.5), fld, cfg)
    assert sorted(p.name for p in tmp_path.glob("*.nsdf")) == ["checkpoint_epoch2.nsdf", "checkpoint_epoch4.nsdf"]
    last = ng.load_model(tmp_path / "checkpoint_epoch4.nsdf")
    np.testing.assert_array_equal(last.Z, work.Z.astype(np.float32))
    rows = log.read_text().strip().splitlines()
    assert rows[0] == "epoch,loss_l1,loss_l2,seconds" and len(rows) == 5


# ------------------------------------------------------------------ model files

def test_model_file_bytes_and_truncation(ng, scenes, golden, tmp_path):
    g = golden("train")
    fld = _tiny(ng, scenes, g, f64=False)
    path = tmp_path / "m.nsdf"
    ng.save_model(path, fld)
    assert path.read_bytes() == g["model_bytes"].tobytes()
    assert ng.serialized_bytes(fld) == int(g["serialized_bytes"])
    ref_path = tmp_path / "ref.nsdf"
    ref_path.write_bytes(g["model_bytes"].tobytes())
    back = ng.load_model(ref_path)
    np.testing.assert_array_equal(back.Z, fld.Z)
    for lv in range(3):
        np.testing.assert_array_equal(back.svo.levels[lv].codes, fld.svo.levels[lv].codes)
    np.testing.assert_array_equal(back.svo.virtual_codes[0], fld.svo.virtual_codes[0])
    pts = g["lb_pts"]
    np.testing.assert_array_equal(back.predict(pts, 2), fld.predict(pts, 2))
    cut = ng.load_model(ref_path, max_lod=1)
    assert cut.svo.corner_count == int(g["cut_corner_count"])
    np.testing.assert_array_equal(cut.svo.region.lo, g["cut_region_lo"])
    np.testing.assert_array_equal(cut.svo.region.hi, g["cut_region_hi"])
    np.testing.assert_array_equal(cut.Z, g["cut_Z"])
    with pytest.raises(ng.ConfigError):
        ng.load_model(ref_path, max_lod=3)
    bad = tmp_path / "bad.nsdf"
    bad.write_bytes(g["model_bytes"].tobytes()[:-3])
    with pytest.raises(ng.FormatError):
        ng.load_model(bad)


def test_device_epoch_sampler_golden(ng, scenes, golden):
    """The GPU surface tracer + device SDF give the reference's epoch set
    (sampling.py:177-196) for the sphere, bit for bit."""
    from paper_2101_10994_b200 import sampling
    g = golden("train")
    ss = sampling.build_epoch_set(scenes.Sphere(0.5), 600, 10)
    np.testing.assert_array_equal(ss.points, g["ep_points"])
    np.testing.assert_array_equal(ss.distances, g["ep_dist"])
    np.testing.assert_array_equal(ss.scheme_tags, g["ep_tags"])


def test_epoch_inputs_copied_asynchronously(ng, scenes, golden):
    """The epoch's next-batch location runs on a side stream: inputs that are
    still being copied (non-blocking from pinned memory) when the epoch is
    enqueued must give the same result as synchronised inputs."""
    import torch
    from paper_2101_10994_b200.trainer import DeviceTrainer
    g = golden("train")
    fld = _tiny(ng, scenes, g)
    rng = np.random.default_rng(21)
    pts = rng.uniform(-0.9, 0.9, size=(5000, 3))
    dist = np.linalg.norm(pts, axis=1) - 0.5
    outs = []
    for asynchronous in (False, True):
        tr = DeviceTrainer(ng.NeuralField(fld.svo, fld.Z.copy(), [d.astype(np.float64) for d in fld.decoders]),
                           256)
        for _ in range(2):
            if asynchronous:
                p = torch.from_numpy(pts).pin_memory().to("cuda", non_blocking=True)
                d = torch.from_numpy(dist).pin_memory().to("cuda", non_blocking=True)
            else:
                p = torch.from_numpy(pts).cuda()
                d = torch.from_numpy(dist).cuda()
                torch.cuda.synchronize()
            tr.run_epoch(p, d, [1, 2], True, 1e-3)
        outs.append(tr.state.Z_numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
