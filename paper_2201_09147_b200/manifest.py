"""Python mirror of the reference's on-disk formats, for tests and bench.py.

  .sdfnet  mlp::save_params / load_params   (src/mlp/io.cpp:15-78): JSON {activation, omega0,
           input_dim, layers[{rows, cols, weights_flat, bias}]}, shortest round-trip doubles.
  .nest    fields::save_manifest / load_manifest (src/fields/manifest.cpp:72-178): JSON
           {time_dependent, deltas, fields[{weights | analytic,params, label}], provenance};
           weight paths resolve relative to the manifest.

The product's own loader is the C++ host library (libnsdf_b200.so); this module only
builds the objects the Python-side API and the tests hand to the C ABI.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .abi import ACT_IDENTITY, ACT_SINE, NsdfError, ERR_PARSE, ERR_VALIDATION, ERR_CONFIG


@dataclass
class Net:
    """MlpParams<double> in the packed layout of nsdf_cuda.h (per layer W row-major, then b)."""
    rows: np.ndarray
    cols: np.ndarray
    packed: np.ndarray
    activation: int = ACT_SINE
    omega0: float = 30.0
    input_dim: int = 3

    @property
    def n_layers(self) -> int:
        return len(self.rows)

    @property
    def width(self) -> int:
        return int(self.rows[0])

    @property
    def hidden_blocks(self) -> int:
        return self.n_layers - 2

    def parameter_count(self) -> int:
        return int(sum(int(r) * int(c) + int(r) for r, c in zip(self.rows, self.cols)))

    def layers(self):
        off = 0
        out = []
        for r, c in zip(self.rows, self.cols):
            r, c = int(r), int(c)
            w = self.packed[off:off + r * c].reshape(r, c)
            off += r * c
            b = self.packed[off:off + r]
            off += r
            out.append((w, b))
        return out

    def macs_forward(self) -> int:
        """MACs per forward eval = d*w + k_h*w^2 + w."""
        return int(sum(int(r) * int(c) for r, c in zip(self.rows, self.cols)))

    def macs_normal(self) -> int:
        """fwd + 3 tangent chains = MACs_fwd + 3*(k_h*w^2 + 2w) + 3w."""
        w = self.width
        return self.macs_forward() + 3 * (self.hidden_blocks * w * w + 2 * w) + 3 * w

    @staticmethod
    def from_layers(layers, activation=ACT_SINE, omega0=30.0, input_dim=3) -> "Net":
        rows = np.array([w.shape[0] for w, _ in layers], np.int32)
        cols = np.array([w.shape[1] for w, _ in layers], np.int32)
        packed = np.concatenate([np.concatenate([np.asarray(w, np.float64).reshape(-1),
                                                 np.asarray(b, np.float64).reshape(-1)]) for w, b in layers])
        return Net(rows, cols, packed, activation, float(omega0), int(input_dim))


@dataclass
class Analytic:
    """Analytic member: sphere {cx,cy,cz,r}, torus {R,r}, box {hx,hy,hz} (field.cpp:375-393)."""
    name: str
    params: dict = field(default_factory=dict)

    def values(self) -> List[float]:
        p = self.params
        if self.name == "sphere":
            return [p.get("cx", 0.0), p.get("cy", 0.0), p.get("cz", 0.0), p.get("r", 0.7)]
        if self.name == "torus":
            return [p.get("R", 0.6), p.get("r", 0.3)]
        if self.name == "box":
            return [p.get("hx", 0.6), p.get("hy", 0.45), p.get("hz", 0.5)]
        raise NsdfError(ERR_CONFIG, f"unknown analytic field '{self.name}' (expected sphere, torus or box)")


@dataclass
class Sequence:
    """NestedSequence / AnimatedSequence (nesting.hpp:53-77)."""
    members: list
    deltas: List[float]
    labels: List[str]
    time_dependent: bool = False
    path: Optional[str] = None
    provenance: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.members)

    def subsequence(self, indices) -> "Sequence":
        return Sequence([self.members[i] for i in indices], [self.deltas[i] for i in indices],
                        [self.labels[i] for i in indices], self.time_dependent, None, self.provenance)


def load_sdfnet(path: str) -> Net:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise NsdfError(ERR_PARSE, f"cannot open weight file {path}") from e
    except json.JSONDecodeError as e:
        raise NsdfError(ERR_PARSE, f"malformed weight file {path}: {e}") from e
    act = {"sine": ACT_SINE, "identity": ACT_IDENTITY}.get(j["activation"])
    if act is None:
        raise NsdfError(ERR_CONFIG, f"unknown activation kind '{j['activation']}'")
    layers = []
    for i, jl in enumerate(j["layers"]):
        r, c = int(jl["rows"]), int(jl["cols"])
        w = np.asarray(jl["weights_flat"], np.float64)
        b = np.asarray(jl["bias"], np.float64)
        if w.size != r * c or b.size != r:
            raise NsdfError(ERR_PARSE, f"layer {i} of {path} has inconsistent weight or bias length")
        layers.append((w.reshape(r, c), b))
    return Net.from_layers(layers, act, float(j["omega0"]), int(j["input_dim"]))


def save_sdfnet(net: Net, path: str) -> None:
    j = {"activation": "sine" if net.activation == ACT_SINE else "identity", "omega0": net.omega0,
         "input_dim": net.input_dim,
         "layers": [{"rows": int(w.shape[0]), "cols": int(w.shape[1]), "weights_flat": w.reshape(-1).tolist(),
                     "bias": b.tolist()} for w, b in net.layers()]}
    with open(path, "w") as f:
        json.dump(j, f, indent=1)


def load_manifest(path: str) -> Sequence:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise NsdfError(ERR_PARSE, f"cannot open manifest {path}") from e
    deltas = [float(d) for d in j["deltas"]]
    fields_ = j["fields"]
    if len(fields_) != len(deltas):
        raise NsdfError(ERR_VALIDATION, f"manifest {path} lists {len(fields_)} fields but {len(deltas)} thresholds")
    td = bool(j.get("time_dependent", False))
    base = os.path.dirname(path)
    members, labels = [], []
    for fe in fields_:
        if "weights" in fe:
            net = load_sdfnet(os.path.join(base, fe["weights"]))
            want = 4 if td else 3
            if net.input_dim != want:
                raise NsdfError(ERR_VALIDATION, f"manifest {path}: {fe['weights']} is not a {want}-input network")
            members.append(net)
        elif "analytic" in fe:
            members.append(Analytic(fe["analytic"], dict(fe.get("params", {}))))
        else:
            raise NsdfError(ERR_PARSE, "manifest field entry has neither 'weights' nor 'analytic'")
        labels.append(fe.get("label", ""))
    return Sequence(members, deltas, labels, td, path, j.get("provenance", {}))


def write_manifest(seq: Sequence, path: str, weight_names: Optional[List[str]] = None) -> None:
    """Write a .nest; analytic members inline, nets by the given relative weight names."""
    fields_ = []
    for i, m in enumerate(seq.members):
        if isinstance(m, Analytic):
            fe = {"analytic": m.name}
            if m.params:
                fe["params"] = m.params
        else:
            fe = {"weights": weight_names[i]}
        if seq.labels[i]:
            fe["label"] = seq.labels[i]
        fields_.append(fe)
    with open(path, "w") as f:
        json.dump({"time_dependent": seq.time_dependent, "deltas": list(seq.deltas), "fields": fields_,
                   "provenance": seq.provenance or {"proposition": 0}}, f, indent=1)
