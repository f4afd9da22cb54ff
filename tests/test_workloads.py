"""Input generators: sizes of BASELINE.json configs (SURVEY.md §8(d) Table D-1),
closed-mesh topology invariants, determinism."""
import numpy as np
import pytest

from workloads import make_mesh, make_vectors, cube_surface, get_config
from workloads.configs import element_layout


@pytest.mark.parametrize("name,N,nt", [("c1", 1152, 768), ("c2", 115200, 76800), ("c3", 526068, 350712),
                                       ("c5", 1119744, 746496)])
def test_config_sizes(name, N, nt):
    m = make_mesh(name)
    assert m.n_rwg == N and m.triangles.shape[0] == nt


@pytest.mark.parametrize("n", [1, 2, 4, 7])
def test_cube_topology(n):
    m = cube_surface((0.1, -0.2, 0.3), 0.4, n)
    V, F, E = m.vertices.shape[0], m.triangles.shape[0], m.rwg.shape[0]
    assert V - E + F == 2 and 2 * E == 3 * F
    # outward winding: signed volume positive
    v = m.vertices[m.triangles]
    vol = np.einsum("ij,ij->i", v[:, 0], np.cross(v[:, 1], v[:, 2])).sum() / 6
    assert abs(vol - 0.4 ** 3) < 1e-12
    # rows sorted by (va, vb), t+ < t-
    r = m.rwg.astype(np.int64)
    key = r[:, 0] * 10 ** 6 + r[:, 1]
    assert (np.diff(key) > 0).all() and (r[:, 2] < r[:, 3]).all()


def test_vectors_deterministic():
    a = make_vectors(100, 3, 0)
    b = make_vectors(100, 3, 0)
    assert a.shape == (100, 3) and np.array_equal(a, b)
    g = np.random.default_rng(0)
    re = g.standard_normal((3, 100))
    assert np.array_equal(a.real, re.T)


def test_c3_sides():
    c, s, n = element_layout(get_config("c3"))
    assert s.min() >= 0.3 and s.max() <= 0.5 and (n == np.ceil(s / 0.05)).all()
