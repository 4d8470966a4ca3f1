import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch, bench
import paper_2101_10994_b200 as ng
knot, samples = bench.knot_scene()
svo = ng.build_octree(knot, 5, samples)
fld = ng.new_field(svo, seed=0)
for n in (20000, 500000):
    t0 = time.perf_counter()
    ss = ng.build_epoch_set(knot, n, 0)
    t1 = time.perf_counter()
    work, hist = ng.train(knot, fld, ng.TrainConfig(epochs=1, points_per_epoch=n, rng_seed=0))
    t2 = time.perf_counter()
    print(n, "sampler s", round(t1 - t0, 3), "train(1 epoch) s", round(t2 - t1, 3), hist[0].level_losses)
