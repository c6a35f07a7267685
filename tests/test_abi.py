"""C-ABI library: loads, exports every symbol include/mra.h declares, host-side plan logic
(no GPU: host-only plans, device = -2). The plan built by the product must agree bit for bit
with the oracle's independent plan."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1905_00141_b200 as mra
import synth
from paper_1905_00141_b200 import build as mbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def lib():
    mbuild.build()
    return mra.load_library()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "mra.h")).read()
    names = set(re.findall(r"^\s*(?:mra_status|uint64_t|void|const char\*)\s+(mra_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 12
    cdll = ctypes.CDLL(mra.LIB_PATH)
    for nme in sorted(names):
        assert hasattr(cdll, nme), nme
    assert names <= set(mra.EXPORTS)


def test_sass_is_sm100a_with_dmma():
    """The library carries sm_100a SASS and its GEMM tiles run on the fp64 tensor path (DMMA)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", mra.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out


@pytest.mark.parametrize("J,M,r,clusters", [(4, 4, 16, 0), (2, 7, 9, 3), (4, 3, 36, 2), (2, 5, 32, 0)])
def test_host_plan_matches_oracle_plan(J, M, r, clusters):
    x, y, _ = synth.uniform_small(3000, seed=J * 10 + M, clusters=clusters, domain=(-5.0, 7.0, 40.0, 41.5))
    p = mra.mra_plan_create(x, y, M, J, r, device=-2)
    lay = mra.mra_plan_layout(p)
    o = oracle.plan(x, y, M, J, r)
    assert p.r_hat == o["r_hat"]
    # knots bit-identical
    np.testing.assert_array_equal(lay["knots_x"].reshape(-1, p.r_hat), o["knots_x"])
    np.testing.assert_array_equal(lay["knots_y"].reshape(-1, p.r_hat), o["knots_y"])
    # leaf assignment: perm/leaf_off reproduce the oracle's leaf of every observation, stable order
    leaf = np.full(len(x), -1)
    off = lay["leaf_off"]
    for l in range(p.n_leaves):
        leaf[lay["perm"][off[l]:off[l + 1]]] = l
        assert np.all(np.diff(lay["perm"][off[l]:off[l + 1]]) > 0)
    np.testing.assert_array_equal(leaf, o["leaf"])
    info = mra.mra_plan_info(p)
    assert info["n_regions"] == (J ** M - 1) // (J - 1)
    assert info["n_empty_leaves"] == int(np.sum(np.diff(off) == 0))
    p.close()


def test_elimination_matches_oracle():
    x, y, z = synth.uniform_small(500, seed=9)
    o = oracle.plan(x, y, 3, 4, 9)
    x2 = np.append(x, [o["knots_x"][1, 3], o["knots_x"][0, 0]])
    y2 = np.append(y, [o["knots_y"][1, 3], o["knots_y"][0, 0]])
    p = mra.mra_plan_create(x2, y2, 3, 4, 9, device=-2)
    assert p.n_retained == 500
    assert set(mra.mra_plan_layout(p)["perm"].tolist()) == set(range(500))


def test_config_and_arg_errors():
    x, y, _ = synth.uniform_small(100, seed=1)
    for args, status in [((3, 3, 16), 2), ((0, 4, 16), 2), ((3, 4, 0), 2), ((3, 4, 100), 2)]:
        with pytest.raises(mra.MraError) as e:
            mra.mra_plan_create(x, y, *args, device=-2)
        assert e.value.status == status
    with pytest.raises(mra.MraError) as e:
        mra.mra_plan_create(np.ones(10), np.arange(10.0), 2, 4, 4, device=-2)
    assert e.value.status == 3                     # degenerate bounding box
    xb = x.copy(); xb[3] = np.nan
    with pytest.raises(mra.MraError) as e:
        mra.mra_plan_create(xb, y, 2, 4, 4, device=-2)
    assert e.value.status == 1
    p = mra.mra_plan_create(x, y, 2, 4, 4, device=-2)
    with pytest.raises(mra.MraError) as e:
        mra.mra_loglik(p, np.zeros(100), (0, 1.0, 0.1, 0.1))
    assert e.value.status == 5                     # host-only plans cannot evaluate (no CPU fallback)


def test_all_eliminated_is_struct_error():
    o = oracle.plan(np.array([0.0, 1.0]), np.array([0.0, 1.0]), 2, 4, 4)
    x = np.append(o["knots_x"][0], [0.0, 1.0]); y = np.append(o["knots_y"][0], [0.0, 1.0])
    # the two extreme points define the same box; knots sit inside -> eliminated, corners stay
    p = mra.mra_plan_create(x, y, 2, 4, 4, device=-2)
    assert p.n_retained == 2


def test_shard_assignment_partitions_subtrees():
    w = synth.make("C4", n=40000)
    owned = []
    for rank in range(4):
        p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, device=-2, rank=rank, world=4)
        s = mra.mra_plan_shards(p)
        owned.append(s["own"])
        lvl = s["shard_level"]
        assert w.J ** (lvl - 1) >= 32
    allv = np.sort(np.concatenate(owned))
    np.testing.assert_array_equal(allv, np.arange(w.J ** (lvl - 1)))


def test_atilde_eq1():
    assert abs(mra.atilde_bound_gib(2, 10, 256) - 11.25) < 1e-12
    assert abs(mra.atilde_bound_gib(2, 14, 49) - 13.34) < 0.005


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors of mra_opts / mra_theta / mra_post have the C layout of include/mra.h
    (field order, offsets, size), checked against gcc's own offsetof."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    structs = {"mra_opts": mra._Opts, "mra_theta": mra._Theta, "mra_post": mra._Post}
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{os.path.join(ROOT, "include", "mra.h")}"',
           "int main(void) {"]
    for cname, py in structs.items():
        src.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            src.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    src += ["return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call([gcc, str(c), "-o", str(exe)])
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, what, v = line.split()
        got[(cname, what)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
    # and every C field is mirrored (no field missing at the end)
    hdr = open(os.path.join(ROOT, "include", "mra.h")).read()
    body = hdr[hdr.index("typedef struct {", hdr.index("Plan options")):hdr.index("} mra_opts;")]
    cfields = re.findall(r"^\s+(?:const\s+)?(?:int|double|void\*)\s+([a-z_0-9, ]+);|^\s+void\*?\s*\(\*([a-z_0-9]+)\)",
                         body, re.M)
    names = [n.strip() for plain, fp in cfields for n in (plain.split(",") if plain else [fp])]
    assert names == [f for f, _ in mra._Opts._fields_]


def test_tree_size_bounds_are_config_errors():
    """an oversized tree is MRA_E_CONFIG before any O(regions) host allocation (no abort)."""
    x, y, _ = synth.uniform_small(100, seed=2)
    for M, J in ((23, 4), (24, 2), (40, 4)):
        with pytest.raises(mra.MraError) as e:
            mra.mra_plan_create(x, y, M, J, 4, device=-2)
        assert e.value.status == 2
    with pytest.raises(mra.MraError) as e:
        mra.mra_plan_create(x, y, 3, 4, 4, device=-2, rank=3, world=2)
    assert e.value.status == 1                     # rank outside [0, world)


def test_nccl_unique_id_without_gpu():
    """The in-library exchange loads NCCL at run time (dlopen); an id can be made on a host without a GPU."""
    a, b = mra.mra_nccl_unique_id(), mra.mra_nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
    with pytest.raises(ValueError):
        mra.mra_plan_create(np.random.rand(10), np.random.rand(10), 2, 4, 4, device=-2, nccl_id=b"short")
    x, y, _ = synth.uniform_small(200, seed=3)
    with pytest.raises(mra.MraError) as e:     # a host-only plan cannot hold a communicator
        mra.mra_plan_create(x, y, 3, 4, 4, device=-2, nccl_id=a)
    assert e.value.status == 1


def test_shard_size_is_packed_lower_triangles():
    """Exchange buffer = per level-s region the packed lower triangle of its q x q output + d, u, + 1 flag."""
    w = synth.make("C1", n=20000)
    p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, device=-2, rank=0, world=2)
    s = mra.mra_plan_shards(p)["shard_level"]
    ns, q = w.J ** (s - 1), (s - 1) * p.r_hat + 1
    assert mra.mra_shard_size(p) == ns * q * (q + 1) // 2 + 2 * ns + 1


def test_shard_assignment_contiguous_on_uniform_data():
    """Uniform leaves (C3 recipe): every rank's subtrees form ONE contiguous run (the smallest-max-load
    contiguous split is within 3 % of LPT there), the runs cover the shard level in rank order."""
    w = synth.make("C3", n=200_000)
    world = 8
    prev_end = 0
    for rank in range(world):
        p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, device=-2, rank=rank, world=world)
        own = mra.mra_plan_shards(p)["own"]
        assert len(own) > 0
        np.testing.assert_array_equal(own, np.arange(own[0], own[0] + len(own)))
        assert own[0] == prev_end
        prev_end = own[-1] + 1
    assert prev_end == w.J ** (mra.mra_plan_shards(p)["shard_level"] - 1)
