"""Runtime behaviour of the boundary (SURVEY.md 8b Threading, ownership):

* concurrent render() calls from two threads, each on its own CUDA stream,
  on different fields and on one field at two LODs (the presummed tables of
  each LOD travel in a per-frame copy of the field struct), equal the same
  frames rendered one after another, bit for bit;
* the reference's training loop pattern forward -> backward -> in-place
  adam_step -> forward sees the updated parameters (device copies of the
  updated arrays are dropped by adam_step).
"""

import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def scenes2():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    go = dict(np.load(os.path.join(ROOT, "tests", "golden", "octree.npz")))
    svo_t = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    torus = scenes.planted_field(svo_t, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
    sph = scenes.Sphere(0.45)
    svo_s = ng.build_octree(sph, 4, scenes.sphere_samples(0.45, 4096, seed=1))
    sphere = scenes.planted_field(svo_s, sph, seed=0)
    cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 200, 150)
    return ng, torus, sphere, cam


def _frame(ng, fld, cam, lod):
    fb, rep = ng.render(cam, fld, ng.RenderConfig(lod=lod))
    return fb.color.copy(), fb.t.copy(), rep.visible, rep.evals


def _threads(ng, jobs, reps=6):
    import torch
    results = {i: [] for i in range(len(jobs))}
    errors = []

    def run(i, fld, cam, lod):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for _ in range(reps):
                    results[i].append(_frame(ng, fld, cam, lod))
            stream.synchronize()
        except Exception as e:  # surfaced below
            errors.append(repr(e))
    th = [threading.Thread(target=run, args=(i,) + j) for i, j in enumerate(jobs)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    return results


def _same(a, b):
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert a[2:] == b[2:]


def test_two_threads_two_fields(scenes2):
    ng, torus, sphere, cam = scenes2
    want = [_frame(ng, torus, cam, None), _frame(ng, sphere, cam, None)]
    got = _threads(ng, [(torus, cam, None), (sphere, cam, None)])
    for i in range(2):
        assert want[i][2] > 100
        for f in got[i]:
            _same(f, want[i])


def test_two_threads_one_field_two_lods(scenes2):
    ng, torus, _, cam = scenes2
    want = [_frame(ng, torus, cam, 4.0), _frame(ng, torus, cam, 3.5)]
    assert want[0][3] != want[1][3]
    got = _threads(ng, [(torus, cam, 4.0), (torus, cam, 3.5)])
    for i in range(2):
        for f in got[i]:
            _same(f, want[i])


def test_forward_adam_forward_sees_updates(scenes2):
    """trainer.py's loop on the public API: forward, backward, adam_step in
    place, forward again -- the second forward must use the new values."""
    ng, torus, _, _ = scenes2
    svo = torus.svo
    fld = ng.NeuralField(svo, np.asarray(torus.Z, np.float64).copy(),
                         [d.astype(np.float64) for d in torus.decoders])
    x = ng.build_epoch_set(__import__("paper_2101_10994_b200").scenes.Torus(0.5, 0.2), 512, 3).points
    out0, cache = fld.forward(x, 3)
    grads = ng.backward(cache, np.ones(len(x)))
    params = {"Z": fld.Z}
    for i, d in enumerate(fld.decoders):
        for k in ("W1", "b1", "W2", "b2"):
            params[f"decoder{i + 1}.{k}"] = getattr(d, k)
    gd = {"Z": grads.dZ}
    for i, g in enumerate(grads.decoders):
        if g is not None:
            for k in ("W1", "b1", "W2", "b2"):
                gd[f"decoder{i + 1}.{k}"] = getattr(g, k)
    ng.adam_step(params, gd, ng.AdamState.for_params(params), 1e-2)
    out1, _ = fld.forward(x, 3)
    fresh = ng.NeuralField(svo, fld.Z.copy(), [ng.Decoder(d.W1.copy(), d.b1.copy(), d.W2.copy(), d.b2.copy())
                                               for d in fld.decoders])
    want, _ = fresh.forward(x, 3)
    assert np.abs(out1 - out0).max() > 1e-4       # the update moved the outputs
    np.testing.assert_array_equal(out1, want)      # and forward sees it
    np.testing.assert_array_equal(fld.predict(x, 3), fresh.predict(x, 3))
