"""PLY / SPL1 formats on the host: header grammar and errors (pcio.py:124-207),
the oracle's body decode pinned to the reference's load_ply / load_splats
outputs (tests/golden/formats), and save_ply writing byte-identical files."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import formats as OF
from paper_2409_16504_b200 import pcio

FMT = GOLDEN / "formats"
META = json.loads((FMT / "formats.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["bin_normals", "bin_plain", "ascii_normals"])
def test_oracle_ply_decode_matches_reference(name):
    pos, col, nrm = OF.read_ply(FMT / f"{name}.ply")
    m = META[name]
    assert sha(pos) == m["positions"] and sha(col) == m["colors"]
    assert (nrm is None and m["normals"] is None) or sha(nrm) == m["normals"]


def test_oracle_spl1_decode_matches_reference():
    d = OF.decode_spl1((FMT / "splats.spl1").read_bytes())
    for k in ("centers", "scales", "quaternions", "opacities", "colors", "normals"):
        assert sha(d[k]) == META["spl1"][k], k


@pytest.mark.parametrize("name,binary", [("bin_normals", True), ("bin_plain", True),
                                         ("ascii_normals", False)])
def test_save_ply_byte_identical(tmp_path, name, binary):
    c = np.load(FMT / "cloud_in.npz")
    nrm = c["normals"] if "normals" in name else None
    out = tmp_path / "x.ply"
    pcio.save_ply(pcio.PointCloud(c["positions"], c["colors"], nrm), out, binary=binary)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == META[name]["file_sha256"]


def header(text: str, tmp_path):
    p = tmp_path / "h.ply"
    p.write_bytes(text.encode("ascii"))
    with open(p, "rb") as fh:
        return pcio._header(fh, str(p))


def test_header_grammar_and_errors(tmp_path):
    ok = ("ply\nformat binary_little_endian 1.0\ncomment x\nelement vertex 3\n"
          "property float x\nproperty float y\nproperty float z\nproperty uchar red\n"
          "property uchar green\nproperty uchar blue\nend_header\n")
    assert header(ok, tmp_path) == (True, 3, ["x", "y", "z", "red", "green", "blue"])
    bad = [("plx\n", pcio.PlyParseError),
           (ok.replace("binary_little_endian", "binary_big_endian"), pcio.PlyUnsupportedError),
           (ok.replace("element vertex 3", "element face 3"), pcio.PlyUnsupportedError),
           (ok.replace("property uchar red", "property float red"), pcio.PlyUnsupportedError),
           (ok.replace("property uchar blue\n", ""), pcio.PlyUnsupportedError),
           (ok.replace("element vertex 3", "element vertex x"), pcio.PlyParseError),
           (ok.replace("end_header\n", ""), pcio.PlyParseError),
           (ok.replace("format binary_little_endian 1.0\n", ""), pcio.PlyParseError)]
    for text, err in bad:
        with pytest.raises(err):
            header(text, tmp_path)
