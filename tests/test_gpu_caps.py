"""The device's fixed capacities where the reference is unbounded: below each
cap the engine equals the oracle, beyond it the ray is flagged MWT_ST_OVERFLOW
(never a silent wrong answer) and the drop-in raises TraversalError.

  kd mailbox   kKdMailbox = 512 distinct primitive tests per ray (accel.py:775 `tested`)
  BVH stack    kBvhStack  = 128 pending nodes (accel.py:492 `stack`)

The structures are built by hand (flattened arrays, as fixtures/gen_fixtures.py
writes them) on the Lines-1024 scene: a one-leaf kd-tree holding P segments,
and a BVH chain of depth D whose every box holds the whole square."""
import numpy as np
import pytest

from conftest import fixture_paths

pytestmark = pytest.mark.gpu


def _one_leaf_kd(p):
    return dict(c_t=np.float64(8.0), num_leaves=np.int64(1), axis=np.array([-1], np.int32),
                pos=np.zeros(1), left=np.array([-1], np.int32), right=np.array([-1], np.int32),
                box=np.array([[0.0, 0.0, 1.0, 1.0]]), ropes=np.full((1, 4), -1, np.int32),
                rope_cost=np.zeros((1, 4), np.int32), prim_off=np.zeros(1, np.int32),
                prim_cnt=np.array([p], np.int32), prims=np.arange(p, dtype=np.int32))


def _bvh_chain(depth):
    # node 2k (k < depth): internal, children leaf 2k+1 and node 2k+2; node 2*depth: leaf
    n = 2 * depth + 1
    left = np.full(n, -1, np.int32)
    right = np.full(n, -1, np.int32)
    for k in range(depth):
        left[2 * k], right[2 * k] = 2 * k + 1, 2 * k + 2
    return dict(c_t=np.float64(1.0), box=np.tile([0.0, 0.0, 1.0, 1.0], (n, 1)), left=left, right=right,
                prim_off=np.zeros(n, np.int32), prim_cnt=np.zeros(n, np.int32),
                prims=np.zeros(0, np.int32))


def _rays():
    from oracle import oracle as orc
    return orc.raygen(1, (0.0, 0.0, 1.0, 1.0), 77, 0, 64)


@pytest.mark.parametrize("p", [500, 512, 513, 600])
def test_kd_mailbox_cap(p):
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceKd, DeviceMesh
    paths = fixture_paths("lines1024", "mwt")
    arrays = _one_leaf_kd(p)
    got = DeviceKd(DeviceMesh.from_files(*paths), arrays).trace(_rays())
    ref = orc.Kd(orc.Mesh.from_files(*paths), arrays).trace(_rays())
    over = (got["status"] & _lib.ST_OVERFLOW) != 0
    if p <= 512:
        assert not over.any()
        for k in ("seg", "nodes", "ropes", "prims"):
            assert np.array_equal(got[k], ref[k]), k
        hit = ref["seg"] >= 0
        assert np.array_equal(got["t"][hit], ref["t"][hit])
    else:
        # every ray tests all p distinct segments of the one leaf before it can stop
        assert over.all() and (ref["prims"] == p).all()


@pytest.mark.parametrize("depth", [100, 127, 128, 140])
def test_bvh_stack_cap(depth):
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceMesh
    paths = fixture_paths("lines1024", "mwt")
    arrays = _bvh_chain(depth)
    got = DeviceBvh(DeviceMesh.from_files(*paths), arrays).trace(_rays())
    ref = orc.Bvh(orc.Mesh.from_files(*paths), arrays).trace(_rays())
    over = (got["status"] & _lib.ST_OVERFLOW) != 0
    # the chain leaves one pending leaf per level: the k-th internal node finds
    # k entries on the stack and needs room for 2 more (k + 2 <= kBvhStack)
    if depth - 1 + 2 <= 128:
        assert not over.any()
        for k in ("seg", "node_tests", "prim_tests"):
            assert np.array_equal(got[k], ref[k]), k
        assert (got["node_tests"] == 1 + 2 * depth).all()
    else:
        assert over.all()


def test_drop_in_raises_where_the_device_overflows(monkeypatch):
    """kd_intersect / bvh_intersect raise TraversalError on an overflowed ray
    (the reference would have answered: the documented divergence)."""
    from paper_2112_05570_b200 import accel
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh
    from paper_2112_05570_b200.geometry import Point, Ray
    mesh = DeviceMesh.from_files(*fixture_paths("lines1024", "mwt"))
    kd = DeviceKd(mesh, _one_leaf_kd(600))
    kd.node_index, kd.is_internal = {}, np.array([False])
    bvh = DeviceBvh(mesh, _bvh_chain(140))
    ray = Ray(Point(0.31, 0.27), Point(0.6, 0.8))

    class Fake:
        scene = None
    monkeypatch.setattr(accel, "_device_struct", lambda obj: obj.dev)
    fk, fb = Fake(), Fake()
    fk.dev, fb.dev = kd, bvh
    with pytest.raises(accel.TraversalError):
        accel.kd_intersect(fk, ray)
    with pytest.raises(accel.TraversalError):
        accel.bvh_intersect(fb, ray)


def _square_fan(k):
    """k triangles fanned from (0.5, 0.5) to k points along the unit square's
    boundary (CCW, corners included): every triangle contains the centre."""
    from paper_2112_05570_b200.formats import SceneArrays, TriArrays
    per = k // 4
    pts = []
    for a, b in (((0, 0), (1, 0)), ((1, 0), (1, 1)), ((1, 1), (0, 1)), ((0, 1), (0, 0))):
        for j in range(per):
            f = j / per
            pts.append((a[0] + (b[0] - a[0]) * f, a[1] + (b[1] - a[1]) * f))
    b = np.array(pts)
    n = len(b)
    vxy = np.vstack([[0.5, 0.5], b])
    v = np.array([[0, 1 + i, 1 + (i + 1) % n] for i in range(n)], np.int32)
    nbr = np.array([[-1, (i + 1) % n, (i - 1) % n] for i in range(n)], np.int32)
    flag = np.array([[i, -1, -1] for i in range(n)], np.int32)
    xy = np.array([[*b[i], *b[(i + 1) % n]] for i in range(n)])
    return SceneArrays(xy, np.ones(n, np.uint8)), TriArrays(vxy, v, nbr, flag)


@pytest.mark.parametrize("k", [100, 160, 164, 200])
def test_locate_flood_cap(k):
    """kFloodCap = 160 triangles in the lowest-id tie flood (accel.py:226-238):
    a point shared by k triangles (a k-triangle fan's centre)."""
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceMesh
    sc, tri = _square_fan(k)
    om = orc.Mesh(orc.RawScene(*(np.ascontiguousarray(sc.xy[:, q]) for q in range(4)), sc.kind),
                  orc.RawTri(np.ascontiguousarray(tri.vxy[:, 0]), np.ascontiguousarray(tri.vxy[:, 1]),
                             tri.v, tri.nbr, tri.flag))
    pts = np.array([[0.5, 0.5], [0.3, 0.2], [0.5, 0.9]])
    rid, rst = om.locate(pts)
    tid, st = DeviceMesh(sc, tri).locate(pts)
    assert np.array_equal(tid[1:], rid[1:])
    if k <= 160:
        assert tid[0] == rid[0] == 0 and not (st[0] & _lib.ST_OVERFLOW)
    else:
        assert rid[0] == 0 and (st[0] & _lib.ST_OVERFLOW)
