"""CPU checks of the drop-in boundary: libsfb200.so loads without a GPU and
exports exactly the entry points include/sfb200.h declares; host-side API
contracts (plans, cameras, options) behave like the reference."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2409_16504_b200 import _lib, netplan, scenes

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "sfb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfb_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_header():
    lib = _lib.load_library()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert lib.sfb_version() >= 2


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_layer_spec_contract():
    with pytest.raises(ValueError, match="odd"):
        netplan.ConvLayerSpec("conv", 2, 3, kernel=2)
    with pytest.raises(ValueError, match="fixed"):
        netplan.ConvLayerSpec("transposed_conv", 2, 3, kernel=3)
    with pytest.raises(ValueError, match="unknown"):
        netplan.ConvLayerSpec("pool", 2, 3)
    assert netplan.ConvLayerSpec("conv", 9, 16).weight_shape == (3, 3, 3, 9, 16)
    specs = netplan.NetworkPlan().layer_specs()
    assert [(s.kind, s.in_channels, s.out_channels) for s in specs][-3:] == \
        [("transposed_conv", 64, 16), ("mlp", 32, 64), ("mlp", 64, 14)]
    with pytest.raises(ValueError, match="decoder"):
        netplan.NetworkPlan((9, 16, 32), (16, 8), 4)


def test_network_weights_validation():
    plan = netplan.NetworkPlan((9, 4, 6), (4,), 5)
    w = netplan.init_random(plan, 0)
    bad = list(w.layers)
    bad[0] = (bad[0][0], bad[0][1][..., :3], bad[0][2])
    with pytest.raises(ValueError, match="weights must be"):
        netplan.NetworkWeights(plan, bad)


def test_scenes_are_deterministic():
    a, va = scenes.config1(n_dirs=500)
    b, vb = scenes.config1(n_dirs=500)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.colors, b.colors)
    assert np.allclose(va[0].rotation @ va[0].rotation.T, np.eye(3))
