import sys, numpy as np
sys.path.insert(0, '.')
import paper_2101_10994_b200 as ng
from oracle import nglod_oracle as O
g = dict(np.load('tests/golden/octree.npz'))
svo = ng.build_octree(O.sdf_sphere(0.5), 3, g['samples_a'])
print("built", [svo.voxel_count(l) for l in range(4)], svo.corner_count)
