"""PLY / SPL1 decoded on the device (sfb_ply_decode / sfb_spl1_*) against the
oracle's numpy decode (itself pinned to the reference, tests/test_formats.py)."""
import hashlib
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import formats as OF
from paper_2409_16504_b200 import pcio
from paper_2409_16504_b200.gaussians import Splats, load_splats, save_splats

pytestmark = pytest.mark.gpu
FMT = GOLDEN / "formats"
META = json.loads((FMT / "formats.json").read_text())


@pytest.mark.parametrize("name", ["bin_normals", "bin_plain", "ascii_normals"])
def test_load_ply_on_device_bit_exact(name):
    cloud = pcio.load_ply(FMT / f"{name}.ply")
    assert cloud.on_device
    pos, col, nrm = OF.read_ply(FMT / f"{name}.ply")
    assert np.array_equal(cloud.positions.cpu().numpy(), pos)
    assert np.array_equal(cloud.colors.cpu().numpy(), col)
    if nrm is None:
        assert cloud.normals is None
    else:
        assert np.array_equal(cloud.normals.cpu().numpy(), nrm)


def test_zero_normal_fallback_and_truncation(tmp_path):
    rng = np.random.default_rng(4)
    pos = rng.normal(size=(50, 3))
    nrm = rng.normal(size=(50, 3))
    nrm[7] = 0.0
    cloud = pcio.PointCloud(pos, rng.random((50, 3)), nrm, validate=False)   # raw rows for the file
    p = tmp_path / "z.ply"
    pcio.save_ply(cloud, p)
    got = pcio.load_ply(p)
    want = OF.read_ply(p)
    assert np.array_equal(got.normals.cpu().numpy(), want[2])
    assert np.array_equal(got.normals[7].cpu().numpy(), [0.0, 0.0, 1.0])
    p.write_bytes(p.read_bytes()[:-5])
    with pytest.raises(pcio.PlyParseError):
        pcio.load_ply(p)


def test_spl1_round_trip_and_reference_bytes(tmp_path):
    d = np.load(FMT / "splats_in.npz")
    sp = Splats(*(d[k] for k in ("centers", "scales", "quaternions", "opacities", "colors",
                                 "normals")), validate=False)
    out = tmp_path / "s.spl1"
    save_splats(out, sp)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == META["spl1"]["file_sha256"]
    back = load_splats(FMT / "splats.spl1")
    ref = OF.decode_spl1((FMT / "splats.spl1").read_bytes())
    for k in ref:
        assert np.array_equal(getattr(back, k).cpu().numpy(), ref[k]), k
    with pytest.raises(ValueError):
        bad = tmp_path / "bad.spl1"
        bad.write_bytes(b"XXXX" + out.read_bytes()[4:])
        load_splats(bad)
