"""The trainer's host data loader (paper_2101_10994_b200.sampling) against
the reference's epoch sample sets (tests/golden/train.npz). CPU only."""

import numpy as np

from paper_2101_10994_b200 import sampling as S
from paper_2101_10994_b200 import scenes


def test_epoch_set_golden(golden):
    g = golden("train")
    ss = S.build_epoch_set(scenes.Sphere(0.5), 600, 10)
    np.testing.assert_array_equal(ss.points, g["ep_points"])
    np.testing.assert_array_equal(ss.distances, g["ep_dist"])
    np.testing.assert_array_equal(ss.scheme_tags, g["ep_tags"])


def test_split_counts_and_dump_roundtrip(tmp_path):
    assert S.split_counts(10) == (4, 4, 2)
    assert S.split_counts(7) == (4, 2, 1)
    ss = S.SampleSet(np.array([[0.1, 0.2, 0.3]]), np.array([0.5]), np.zeros(1, np.int8))
    S.dump_samples(tmp_path / "s.bin", ss)
    back = S.load_samples(tmp_path / "s.bin")
    np.testing.assert_allclose(back.points, ss.points.astype(np.float32))
    assert back.scheme_tags[0] == S.SCHEME_UNIFORM


def test_mesh_surface_sampler_matches_reference(reference):
    """sample_surface_mesh (sampling.py:50-63) on a reference TriangleMesh:
    the same points, bit for bit (same generator call order)."""
    from paper_2101_10994_b200.sampling import sample_surface_mesh
    sampling = __import__("octfield.sampling", fromlist=["x"])
    geometry = __import__("octfield.geometry", fromlist=["x"])
    v = np.array([[0, 0, 0], [0.5, 0, 0], [0, 0.5, 0], [0, 0, 0.5]], dtype=np.float64)
    f = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    mesh = geometry.TriangleMesh(v, f)
    a = sampling.sample_surface_mesh(mesh, 4096, 11)
    b = sample_surface_mesh(mesh, 4096, 11)
    assert np.array_equal(a, b)
