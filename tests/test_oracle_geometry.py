"""Pins for the input generator and the oracle's element geometry (O-geom).

Pinned against closed-form mesh counts, the measure of the domain,
partition of unity of the P1 gradients, the exact gradient of
linear fields, and a hand-computed unit element.  None of these retypes the oracle.
"""
import numpy as np
import pytest

import fem_inputs as fi


def test_mesh_counts():
    m = fi.grid_tri3(2, 2)
    assert (m.n_nodes, m.n_elems) == (9, 8)
    t = fi.grid_tet4(1, 1, 1)
    assert (t.n_nodes, t.n_elems) == (8, 6)                      # SPEC S:53 (6 tets/cell)
    c1 = fi.config_mesh(1)
    assert (c1.n_nodes, c1.n_elems, c1.n_u) == (81, 128, 162)   # BASELINE cfg 1


@pytest.mark.parametrize("mesh", [fi.perturb(fi.grid_tri3(9, 7), 0.2, 3),
                                  fi.perturb(fi.grid_tet4(4, 3, 5), 0.1, 4),
                                  fi.delaunay_tri3(300, 10, 3), fi.delaunay_tet4(400, 5, 3)])
def test_generator_orientation_positive(mesh):
    x = mesh.coords[mesh.conn]
    J = np.stack([x[:, a] - x[:, 0] for a in range(1, mesh.dim + 1)], axis=2)
    assert np.all(np.linalg.det(J) > 0)


def test_delaunay_tet4_is_a_conforming_tiling_with_irregular_degrees():
    """The unstructured 3D mesh (App. A's general tets): conforming (every face shared
    by <= 2 tets), boundary triangles exactly tile the 6 cube faces (area 6), interior node
    degrees irregular and above 16 for some nodes (the fallback paths of the GPU gathers)."""
    m = fi.delaunay_tet4(600, 5, 1)
    faces = np.sort(np.concatenate([m.conn[:, [0, 1, 2]], m.conn[:, [0, 1, 3]],
                                    m.conn[:, [0, 2, 3]], m.conn[:, [1, 2, 3]]]), axis=1)
    uf, cnt = np.unique(faces, axis=0, return_counts=True)
    assert set(cnt.tolist()) <= {1, 2}
    b = m.coords[uf[cnt == 1]]                                   # [nb, 3 nodes, 3]
    area = 0.5 * np.linalg.norm(np.cross(b[:, 1] - b[:, 0], b[:, 2] - b[:, 0]), axis=1)
    assert abs(area.sum() - 6.0) < 1e-12
    assert np.all([(np.ptp(t, axis=0) < 1e-15).any() for t in b])   # each lies in a face plane
    adj = [set() for _ in range(m.n_nodes)]
    for e in m.conn:
        for a in e:
            adj[a].update(e)
    deg = np.array([len(s) - 1 for s in adj])
    assert deg.max() > 16 and deg.min() < 14


def test_kuhn_split_is_conforming():
    # every interior face of a conforming tet mesh is shared by exactly 2 tets
    m = fi.grid_tet4(3, 3, 3)
    faces = np.sort(np.concatenate([m.conn[:, [0, 1, 2]], m.conn[:, [0, 1, 3]],
                                    m.conn[:, [0, 2, 3]], m.conn[:, [1, 2, 3]]]), axis=1)
    _, cnt = np.unique(faces, axis=0, return_counts=True)
    assert set(cnt.tolist()) <= {1, 2}
    assert np.sum(cnt == 1) == 6 * 2 * 9          # boundary triangles: 6 faces x 2 x 3^2


@pytest.mark.parametrize("mesh,measure", [(fi.perturb(fi.grid_tri3(8, 8), 0.2, 11), 1.0),
                                          (fi.perturb(fi.grid_tet4(5, 4, 3), 0.1, 5), 1.0),
                                          (fi.delaunay_tet4(400, 5, 3), 1.0)])
def test_volume_sum_and_partition_of_unity(oracle_mod, mesh, measure):
    G, vol = oracle_mod.Oracle(mesh).geometry()
    assert np.all(vol > 0)
    assert abs(vol.sum() - measure) < 1e-14
    assert np.abs(G.sum(axis=1)).max() < 1e-12 * np.abs(G).max()   # sum_a G_a = 0


@pytest.mark.parametrize("mesh", [fi.perturb(fi.grid_tri3(6, 5), 0.2, 2),
                                  fi.perturb(fi.grid_tet4(3, 3, 3), 0.1, 2),
                                  fi.delaunay_tet4(100, 3, 2)])
def test_gradient_of_linear_fields_is_exact(oracle_mod, mesh):
    # sum_a x_a (x) G_a = I for the identity map, and = A for u = A x
    G, _ = oracle_mod.Oracle(mesh).geometry()
    x = mesh.coords[mesh.conn]                                   # [E, nen, d]
    eye = np.einsum("eai,eaj->eij", x, G)
    assert np.abs(eye - np.eye(mesh.dim)).max() < 1e-11


def test_unit_right_triangle_and_tet(oracle_mod):
    tri = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                  conn=np.array([[0, 1, 2]], np.int32))
    G, vol = oracle_mod.Oracle(tri).geometry()
    assert vol[0] == 0.5                                          # detJ = 1
    assert np.array_equal(G[0], np.array([[-1., -1.], [1., 0.], [0., 1.]]))
    tet = fi.Mesh(dim=3, coords=np.array([[0., 0., 0.], [1., 0., 0.], [0., 1., 0.], [0., 0., 1.]]),
                  conn=np.array([[0, 1, 2, 3]], np.int32))
    G, vol = oracle_mod.Oracle(tet).geometry()
    assert vol[0] == 1.0 / 6.0
    assert np.array_equal(G[0], np.array([[-1., -1., -1.], [1., 0., 0.], [0., 1., 0.], [0., 0., 1.]]))


def test_degenerate_element_rejected(oracle_mod):
    tri = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [2., 0.]]),
                  conn=np.array([[0, 1, 2]], np.int32))
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.Oracle(tri).geometry()
    assert ei.value.status == 2
    flipped = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                      conn=np.array([[0, 2, 1]], np.int32))
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Oracle(flipped).energy(np.zeros(6))
