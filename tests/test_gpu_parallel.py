"""Multi-rank frames on real renders, two ranks sharing the
one GPU of the test box over gloo (NG_DIST_BACKEND=gloo is what bench.py
uses for the same purpose): TiledRenderer's banded frame, gathered to rank
0 and to all ranks, equals the single-rank render() bit for bit in every
gathered output (colour, depth, hit, normals, iterations); the same holds
when one rank's first attempt overflows its workspace and the ranks agree
on a rerun; and `bench.py --gpus 2` launches its own two ranks and prints
one line with n_gpus = 2.
"""

import json
import os
import signal
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("color", "t", "hit", "normal", "iterations", "evals")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import paper_2101_10994_b200 as ng
    from paper_2101_10994_b200 import scenes
    from oracle import nglod_oracle as O
    go = dict(np.load(os.path.join(ROOT, "tests", "golden", "octree.npz")))
    svo = ng.build_octree(O.sdf_torus(0.5, 0.2), 4, go["samples_b"])
    fld = scenes.planted_field(svo, O.sdf_torus(0.5, 0.2), seed=0, device_sdf=False)
    cam = ng.Camera((0.0, 2.0, 3.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 30.0, 160, 117)
    return ng, fld, cam


def _batch_cams(ng, cam):
    return [cam, ng.Camera((2.5, 2.0, 2.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 35.0, cam.width, cam.height),
            ng.Camera((-1.0, -2.5, 2.5), (0.1, 0.0, 0.0), (0.0, 0.0, 1.0), 40.0, cam.width, cam.height)]


def _worker(rank, world, port, tiny_rank, q, batch=False):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ng, fld, cam = _scene()
        from paper_2101_10994_b200.parallel import TiledRenderer
        if batch:  # three cameras per launch, every frame's tiles in one collective per field
            tiles = TiledRenderer(fld, cam.width, cam.height, batch=3)
            to0, vis, ev = tiles.render_batch(_batch_cams(ng, cam), ng.RenderConfig(), fields=FIELDS, dst=0)
            out = {"rank": rank, "n_visible": vis, "n_evals": ev, "dst_keys": sorted(to0)}
            if rank == 0:
                out.update({k: v.cpu().numpy() for k, v in to0.items()})
            q.put(out)
            dist.destroy_process_group()
            return
        tiles = TiledRenderer(fld, cam.width, cam.height)
        if rank == tiny_rank:  # this rank's first attempt overflows its pair buffers
            tiles.sess.pair_cap = 64
            tiles.sess.hit_cap = 64
            tiles.sess._alloc_ws()
        to0, vis, ev = tiles.render(cam, ng.RenderConfig(), fields=FIELDS, dst=0)
        reruns = tiles.reruns
        everyone, _, _ = tiles.render(cam, ng.RenderConfig(), fields=("color", "t"))
        out = {"rank": rank, "n_visible": vis, "n_evals": ev, "reruns": reruns, "dst_keys": sorted(to0)}
        if rank == 0:
            out.update({k: v.cpu().numpy() for k, v in to0.items()})
        out["all_color"] = everyone["color"].cpu().numpy()
        out["all_t"] = everyone["t"].cpu().numpy()
        q.put(out)
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put({"rank": rank, "error": traceback.format_exc() + repr(e)})


def _run(world, tiny_rank=-1, batch=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tiny_rank, q, batch)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        o = q.get(timeout=300)
        got[o["rank"]] = o
    for p in procs:
        p.join(timeout=60)
    for o in got.values():
        assert "error" not in o, o.get("error")
    return got


@pytest.fixture(scope="module")
def single():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ng, fld, cam = _scene()
    fb, rep = ng.render(cam, fld, ng.RenderConfig())
    return {"color": fb.color, "t": fb.t, "hit": fb.hit, "normal": fb.normal, "iterations": fb.iterations,
            "evals": fb.evals, "visible": rep.visible, "n_evals": rep.evals}


def _same(got, single, names):
    for k in names:
        a, b = np.asarray(got[k]), np.asarray(single[k])
        if k == "hit":
            a = a.astype(bool)
        np.testing.assert_array_equal(a.reshape(b.shape), b, err_msg=k)


@pytest.mark.parametrize("world", [2, 3])
def test_banded_frame_equals_single_rank(single, world):
    got = _run(world)
    r0 = got[0]
    assert r0["dst_keys"] == sorted(FIELDS)
    assert all(got[r]["dst_keys"] == [] for r in range(1, world))  # gathered to rank 0 only
    _same(r0, single, FIELDS)
    for r in range(world):
        assert got[r]["n_visible"] == single["visible"] and got[r]["n_evals"] == single["n_evals"]
        _same({"color": got[r]["all_color"], "t": got[r]["all_t"]}, single, ("color", "t"))


def test_banded_batch_equals_render():
    """Two ranks render three cameras as one batch each (their bands of every frame in one launch
    sequence), gathered to rank 0 as (3, H, W, ...): every frame equals render() for its camera."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ng, fld, cam = _scene()
    cams = _batch_cams(ng, cam)
    want = [ng.render(c, fld, ng.RenderConfig()) for c in cams]
    got = _run(2, batch=True)
    r0 = got[0]
    assert r0["dst_keys"] == sorted(FIELDS) and got[1]["dst_keys"] == []
    for f, (fb, rep) in enumerate(want):
        single = {k: getattr(fb, k) for k in FIELDS}
        _same({k: r0[k][f] for k in FIELDS}, single, FIELDS)
    assert got[0]["n_visible"] == got[1]["n_visible"] == sum(r.visible for _, r in want)


def test_overflow_on_one_rank_reruns_all(single):
    got = _run(2, tiny_rank=1)
    assert got[0]["reruns"] >= 1 and got[1]["reruns"] == got[0]["reruns"]
    _same(got[0], single, FIELDS)


def test_bench_spawns_its_ranks():
    """`bench.py --gpus 2` without torchrun variables starts two ranks
    (here on one GPU over gloo) and prints one line with n_gpus = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["NG_DIST_BACKEND"] = "gloo"
    env["PYTHONFAULTHANDLER"] = "1"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--no-query", "--no-cpu", "--no-extra", "--no-train"]
    # (the run takes ~10 s; a launch that never got past the rendezvous on a
    # busy box is retried once, on a fresh port, before it counts)
    for attempt in range(2):
        p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env, cwd=ROOT,
                             start_new_session=True)  # (its own process group: the ranks go with it)
        try:
            out, err = p.communicate(timeout=150)
            r = subprocess.CompletedProcess(cmd, p.returncode, out, err)
            break
        except subprocess.TimeoutExpired:
            os.killpg(p.pid, signal.SIGABRT)  # the ranks dump their Python stacks (faulthandler)
            out, err = p.communicate()
            msg = ("bench.py --gpus 2 timed out\n" + out[-2000:] + "\n" +
                   "\n".join(ln for ln in err.splitlines() if "NCCL INFO" not in ln)[-6000:])
            if attempt == 1:
                raise AssertionError(msg)
            print(msg, file=sys.stderr)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"].startswith("tiles2")
    assert line["frame"]["visible"] == 112420
