"""P2ENet topology, weights and the P2EN weight-file format (host side).

Mirrors the reference's network description so weights interoperate
bit-for-bit: ``ConvLayerSpec``/``NetworkPlan`` (sparsenet.py:39-118),
``NetworkWeights`` (121-147), ``init_random`` (150-159) and the P2EN file
(save_weights 344-365, load_weights 390-434, layout SPEC.md:410). The device
side packs these into the per-layer GEMM operands in ``sparsenet.py``.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

WEIGHT_MAGIC = b"P2EN"
WEIGHT_VERSION = 1
HEAD_CHANNELS = 14

KIND_CODE = {"conv": 0, "transposed_conv": 1, "mlp": 2}
KIND_NAME = {v: k for k, v in KIND_CODE.items()}
_DEFAULT_KERNEL_STRIDE = {"conv": (3, 1), "transposed_conv": (2, 2), "mlp": (1, 1)}


class WeightFormatError(ValueError):
    """Weight file with a bad magic, version, or layer-kind byte."""


class WeightTruncationError(WeightFormatError):
    """Weight file that ends before its own headers say it should."""


class WeightShapeError(WeightFormatError):
    """Weight file whose sizes or topology disagree with its metadata."""


@dataclass(frozen=True)
class ConvLayerSpec:
    """One layer: conv (odd kernel, stride 1), transposed_conv (2, 2) or mlp (1, 1)."""

    kind: str
    in_channels: int
    out_channels: int
    kernel: int = None
    stride: int = None

    def __post_init__(self):
        if self.kind not in KIND_CODE:
            raise ValueError(f"unknown layer kind '{self.kind}'")
        if self.in_channels <= 0 or self.out_channels <= 0:
            raise ValueError("channel counts must be positive")
        k0, s0 = _DEFAULT_KERNEL_STRIDE[self.kind]
        if self.kernel is None:
            object.__setattr__(self, "kernel", k0)
        if self.stride is None:
            object.__setattr__(self, "stride", s0)
        if self.kind == "conv" and (self.kernel < 1 or self.kernel % 2 == 0):
            raise ValueError(f"conv kernels must be odd, got {self.kernel}")
        if self.kind != "conv" and self.kernel != k0:
            raise ValueError(f"{self.kind} kernel is fixed at {k0}")
        if self.stride != s0:
            raise ValueError(f"{self.kind} stride is fixed at {s0}")

    @property
    def weight_shape(self) -> tuple:
        """(k,k,k,in,out) tap-major; tap [a,b,c] is offset (dz,dy,dx) = (a-r,b-r,c-r)."""
        if self.kind == "mlp":
            return (self.in_channels, self.out_channels)
        k = self.kernel
        return (k, k, k, self.in_channels, self.out_channels)

    @property
    def taps(self) -> int:
        return 1 if self.kind == "mlp" else self.kernel ** 3


@dataclass(frozen=True)
class NetworkPlan:
    """Encoder widths (first = input width), decoder widths (deepest first), head width."""

    encoder_channels: tuple = (9, 16, 32, 64, 128)
    decoder_channels: tuple = (64, 32, 16)
    head_hidden: int = 64

    def __post_init__(self):
        object.__setattr__(self, "encoder_channels", tuple(int(c) for c in self.encoder_channels))
        object.__setattr__(self, "decoder_channels", tuple(int(c) for c in self.decoder_channels))
        if len(self.encoder_channels) < 3:
            raise ValueError("encoder needs an input width, one level, and a bottleneck")
        if len(self.decoder_channels) != self.levels:
            raise ValueError(
                f"decoder must have {self.levels} stages to mirror the encoder, "
                f"got {len(self.decoder_channels)}")
        if any(c <= 0 for c in self.encoder_channels + self.decoder_channels):
            raise ValueError("channel widths must be positive")
        if self.head_hidden <= 0:
            raise ValueError("head width must be positive")

    @property
    def levels(self) -> int:
        return len(self.encoder_channels) - 2

    def layer_specs(self) -> list:
        """Forward order: encoder convs, decoder transposed convs, 2 head MLPs."""
        enc = self.encoder_channels
        out = [ConvLayerSpec("conv", a, b) for a, b in zip(enc[:-1], enc[1:])]
        width = enc[-1]
        for cout, skip in zip(self.decoder_channels, enc[-2:0:-1]):
            out.append(ConvLayerSpec("transposed_conv", width, cout))
            width = cout + skip
        out.append(ConvLayerSpec("mlp", width, self.head_hidden))
        out.append(ConvLayerSpec("mlp", self.head_hidden, HEAD_CHANNELS))
        return out


@dataclass(eq=False)
class NetworkWeights:
    """Plan plus (spec, float32 weights, float32 bias) per layer, forward order."""

    plan: NetworkPlan
    layers: list

    def __post_init__(self):
        want = self.plan.layer_specs()
        if len(self.layers) != len(want):
            raise ValueError(f"plan expects {len(want)} layers, got {len(self.layers)}")
        checked = []
        for i, ((spec, w, b), ref) in enumerate(zip(self.layers, want)):
            if spec != ref:
                raise ValueError(f"layer {i} is {spec}, plan expects {ref}")
            w = np.ascontiguousarray(w, dtype=np.float32)
            b = np.ascontiguousarray(b, dtype=np.float32)
            if w.shape != spec.weight_shape:
                raise ValueError(f"layer {i} weights must be {spec.weight_shape}, got {w.shape}")
            if b.shape != (spec.out_channels,):
                raise ValueError(f"layer {i} bias must be ({spec.out_channels},), got {b.shape}")
            checked.append((spec, w, b))
        self.layers = checked

    def as_oracle_layers(self) -> list:
        """Plain dicts for the CPU oracle (tests only)."""
        return [dict(kind=s.kind, kernel=s.kernel, cin=s.in_channels, cout=s.out_channels,
                     w=w, b=b) for s, w, b in self.layers]


def init_random(plan: NetworkPlan, seed: int) -> NetworkWeights:
    """U(+-sqrt(6/fan_in)) float32 weights, zero biases, one default_rng stream
    consumed in layer order (sparsenet.py:150-159) — bit-identical weights."""
    rng = np.random.default_rng(seed)
    layers = []
    for spec in plan.layer_specs():
        fan_in = spec.in_channels * (1 if spec.kind == "mlp" else spec.kernel ** 3)
        bound = np.sqrt(6.0 / fan_in)
        w = rng.uniform(-bound, bound, size=spec.weight_shape).astype(np.float32)
        layers.append((spec, w, np.zeros(spec.out_channels, dtype=np.float32)))
    return NetworkWeights(plan, layers)


def weights_to_bytes(weights: NetworkWeights) -> bytes:
    """P2EN blob: magic, u32 version, u32 levels, u32-counted channel lists,
    u32 head width, u32 layer count, then per layer u8 kind, u8 kernel, u32 in,
    u32 out, f32 weights (tap-lexicographic), f32 bias; little-endian."""
    plan = weights.plan
    blob = [WEIGHT_MAGIC, struct.pack("<II", WEIGHT_VERSION, plan.levels)]
    for ch in (plan.encoder_channels, plan.decoder_channels):
        blob.append(struct.pack(f"<I{len(ch)}I", len(ch), *ch))
    blob.append(struct.pack("<II", plan.head_hidden, len(weights.layers)))
    for spec, w, b in weights.layers:
        blob.append(struct.pack("<BBII", KIND_CODE[spec.kind], spec.kernel,
                                spec.in_channels, spec.out_channels))
        blob.append(np.ascontiguousarray(w, dtype="<f4").tobytes())
        blob.append(np.ascontiguousarray(b, dtype="<f4").tobytes())
    return b"".join(blob)


def save_weights(weights: NetworkWeights, path) -> None:
    try:
        with open(path, "wb") as fh:
            fh.write(weights_to_bytes(weights))
    except OSError as exc:
        raise OSError(f"cannot write weights {path}: {exc}") from exc


def weights_from_bytes(blob: bytes, path="<bytes>") -> NetworkWeights:
    """Parse and validate a P2EN blob (sparsenet.py:390-434 error contract)."""
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(blob):
            raise WeightTruncationError(f"{path}: file ends inside a field")
        pos += n
        return blob[pos - n:pos]

    def u32(n=1):
        return struct.unpack(f"<{n}I", take(4 * n))

    if take(4) != WEIGHT_MAGIC:
        raise WeightFormatError(f"{path}: not a weight file (bad magic)")
    (version,) = u32()
    if version != WEIGHT_VERSION:
        raise WeightFormatError(f"{path}: unsupported version {version}")
    (levels,) = u32()
    (ne,) = u32()
    enc = u32(ne)
    (nd,) = u32()
    dec = u32(nd)
    head, count = u32(2)
    try:
        plan = NetworkPlan(enc, dec, head)
    except ValueError as exc:
        raise WeightShapeError(f"{path}: {exc}") from exc
    if plan.levels != levels:
        raise WeightShapeError(f"{path}: header says {levels} levels, plan has {plan.levels}")
    layers = []
    for i in range(count):
        kind, kernel = struct.unpack("<BB", take(2))
        cin, cout = u32(2)
        if kind not in KIND_NAME:
            raise WeightFormatError(f"{path}: layer {i} has unknown kind byte {kind}")
        try:
            spec = ConvLayerSpec(KIND_NAME[kind], cin, cout, kernel=kernel)
        except ValueError as exc:
            raise WeightShapeError(f"{path}: layer {i}: {exc}") from exc
        nw = int(np.prod(spec.weight_shape))
        w = np.frombuffer(take(4 * nw), dtype="<f4").reshape(spec.weight_shape).astype(np.float32)
        b = np.frombuffer(take(4 * cout), dtype="<f4").astype(np.float32)
        layers.append((spec, w, b))
    if pos != len(blob):
        raise WeightShapeError(f"{path}: {len(blob) - pos} trailing bytes after last layer")
    try:
        return NetworkWeights(plan, layers)
    except ValueError as exc:
        raise WeightShapeError(f"{path}: {exc}") from exc


def load_weights(path) -> NetworkWeights:
    try:
        with open(path, "rb") as fh:
            blob = fh.read()
    except OSError as exc:
        raise OSError(f"cannot read weights {path}: {exc}") from exc
    return weights_from_bytes(blob, path)
