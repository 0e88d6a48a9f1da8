"""Experiment harness: tensor generation / MXT1 ingestion, sweeps, JSON / CSV reports.

The reference specifies this caller but does not ship it (SPEC.md:347-400,
module ``harness_cli``; SURVEY §8 f, rank 3).  It sits on the caller side of
the hot path: every sweep point runs the fused GPU forward (``dma_attention``)
-- or, with ``target="scores"``, the GPU ``mixed_precision_scores`` -- against
the full-precision ``reference_attention`` / ``reference_scores`` computed
once per input head, and emits one flat ``MetricReport`` row per
(sweep point, head) in sweep order.  There is no CPU fallback: without a
CUDA device ``run_experiment`` raises like every other compute entry point.

  python -m paper_2604_03950_b200.harness --seq-len 1024 --head-dim 64 --heads 2 \\
      --format mxfp8 nvfp4 mxfp4 --diag 0 128 --sink 0 128 --report json --out r.json

TensorFile: little-endian, ``b"MXT1"``, u32 dtype
(0 = f32, the only one), u32 ndim, ndim x u32 dims, then prod(dims) f32
values row-major.
"""

from __future__ import annotations

import argparse
import csv
import io
import itertools
import json
import math
import os
import struct
import sys
from dataclasses import dataclass, field

import numpy as np

MXT1_MAGIC = b"MXT1"
MXT1_F32 = 0


class TensorFileError(ValueError):
    """Malformed or inconsistent MXT1 input; the message names the path and field."""


# ------------------------------------------------------------------ MXT1 files
def write_tensor(path: str, x) -> None:
    """Write ``x`` (any real array) as an MXT1 f32 tensor file."""
    a = np.ascontiguousarray(np.asarray(x, dtype="<f4"))
    if a.ndim < 1:
        raise TensorFileError(f"{path}: a tensor file needs ndim >= 1")
    with open(path, "wb") as f:
        f.write(MXT1_MAGIC + struct.pack("<II", MXT1_F32, a.ndim) + struct.pack(f"<{a.ndim}I", *a.shape))
        f.write(a.tobytes())


def read_tensor(path: str) -> np.ndarray:
    """Read an MXT1 file into a float32 array (errors name the path and the offending field)."""
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path}: no such tensor file")
    with open(path, "rb") as f:
        buf = f.read()
    if len(buf) < 12:
        raise TensorFileError(f"{path}: truncated header ({len(buf)} bytes, need >= 12)")
    if buf[:4] != MXT1_MAGIC:
        raise TensorFileError(f"{path}: bad magic {buf[:4]!r} (expected {MXT1_MAGIC!r})")
    dtype, ndim = struct.unpack_from("<II", buf, 4)
    if dtype != MXT1_F32:
        raise TensorFileError(f"{path}: unsupported dtype code {dtype} (0 = f32 is the only one)")
    if ndim < 1 or ndim > 8:
        raise TensorFileError(f"{path}: bad ndim {ndim}")
    hdr = 12 + 4 * ndim
    if len(buf) < hdr:
        raise TensorFileError(f"{path}: truncated dims (ndim {ndim})")
    dims = struct.unpack_from(f"<{ndim}I", buf, 12)
    n = math.prod(dims)
    if len(buf) - hdr != 4 * n:
        raise TensorFileError(f"{path}: payload is {len(buf) - hdr} bytes, dims {list(dims)} need {4 * n}")
    return np.frombuffer(buf, dtype="<f4", offset=hdr, count=n).reshape(dims).astype(np.float32)


# ------------------------------------------------------------ seeded tensors
def _splitmix64(state: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 counter array (wrap-around arithmetic)."""
    z = state + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _normals(seed: int, stream: int, n: int) -> np.ndarray:
    """n standard normals: Box-Muller (cosine branch) on two splitmix64 uniforms per value.

    Value i uses counters c = 2 i, 2 i + 1 of stream ``stream``: u = (splitmix64(seed * 2^32 +
    stream * 2^40 + c) >> 11) * 2^-53, u1 moved into (0, 1]; z = sqrt(-2 ln u1) cos(2 pi u2).
    """
    with np.errstate(over="ignore"):
        base = np.uint64((seed * (1 << 32) + stream * (1 << 40)) % (1 << 64))
        c = np.arange(2 * n, dtype=np.uint64) + base
        u = (_splitmix64(c) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u1, u2 = 1.0 - u[0::2], u[1::2]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def generate_tensors(len_q: int, len_k: int, dim: int, heads: int, seed: int, stddev: float = 1.0):
    """Deterministic Gaussian Q [heads, len_q, dim], K, V [heads, len_k, dim] (float32).

    SPEC.md:375-382.  Streams 0 / 1 / 2 of ``_normals`` for Q / K / V, scaled by
    ``stddev`` and rounded to float32 (the tensor-file precision).
    """
    for name, val in (("len_q", len_q), ("len_k", len_k), ("dim", dim), ("heads", heads)):
        if int(val) < 1:
            raise ValueError(f"{name} must be positive (got {val})")
    shapes = ((heads, len_q, dim), (heads, len_k, dim), (heads, len_k, dim))
    return tuple((_normals(seed, s, math.prod(sh)) * stddev).astype(np.float32).reshape(sh)
                 for s, sh in enumerate(shapes))


# ------------------------------------------------------------------- configs
FORMAT_NAMES = ("mxfp8", "nvfp4", "mxfp4", "identity")
GRANULARITY_NAMES = ("token", "tensor", "block")


@dataclass
class RunConfig:
    """one input source, attention settings, sweep axes, output."""

    seq_len: int = 1024
    seq_len_k: int | None = None
    head_dim: int = 64
    heads: int = 1
    seed: int = 0
    stddev: float = 1.0
    q_path: str | None = None
    k_path: str | None = None
    v_path: str | None = None
    formats: list = field(default_factory=lambda: ["nvfp4"])
    diag: list = field(default_factory=lambda: [128])
    sink: list = field(default_factory=lambda: [128])
    granularity: list = field(default_factory=lambda: ["token"])
    causal: bool = True
    tile_m: int = 128
    tile_n: int = 128
    pv_mode: str = "mxfp8"
    target: str = "output"  # "output" (final O) or "scores" (post-softmax probabilities)
    out: str | None = None
    report: str = "json"

    def validate(self):
        files = [p is not None for p in (self.q_path, self.k_path, self.v_path)]
        if any(files) and not all(files):
            raise ValueError("tensor-file input needs all of --q, --k and --v")
        for f in self.formats:
            if f not in FORMAT_NAMES:
                raise ValueError(f"unknown format {f!r} (one of {FORMAT_NAMES})")
        for g in self.granularity:
            if g not in GRANULARITY_NAMES:
                raise ValueError(f"unknown granularity {g!r} (one of {GRANULARITY_NAMES})")
        if self.target not in ("output", "scores"):
            raise ValueError("target must be 'output' or 'scores'")
        if self.report not in ("json", "csv"):
            raise ValueError("report must be 'json' or 'csv'")
        if not (self.formats and self.diag and self.sink and self.granularity):
            raise ValueError("every sweep axis needs at least one value")

    def points(self):
        """The sweep product in emission order: format, diag, sink, granularity."""
        return list(itertools.product(self.formats, self.diag, self.sink, self.granularity))


def attention_config(cfg: RunConfig, fmt: str, diag: int, sink: int, gran: str):
    """Map one sweep point to an ``AttentionConfig`` (the named format is the LOW path; the
    high path is MXFP8 E4M3; ``identity`` disables quantization on both paths)."""
    from . import formats as F
    from .attention import AttentionConfig
    from .quantize import Granularity

    low = {"mxfp8": F.MXFP8_E4M3, "nvfp4": F.NVFP4, "mxfp4": F.MXFP4, "identity": None}[fmt]
    high = None if fmt == "identity" else F.MXFP8_E4M3
    return AttentionConfig(tile_m=cfg.tile_m, tile_n=cfg.tile_n, diag_window=diag, sink_window=sink,
                           causal=cfg.causal, low_format=low, high_format=high,
                           granularity=Granularity[gran.upper()], pv_mode=cfg.pv_mode)


def load_inputs(cfg: RunConfig):
    """Q, K, V as float32 [heads, L, D] arrays, from files or the seeded generator."""
    if cfg.q_path is not None:
        q, k, v = (read_tensor(p) for p in (cfg.q_path, cfg.k_path, cfg.v_path))
        for p, x in zip((cfg.q_path, cfg.k_path, cfg.v_path), (q, k, v)):
            if x.ndim not in (2, 3):
                raise TensorFileError(f"{p}: dims {list(x.shape)}: expected [L, D] or [heads, L, D]")
        q, k, v = (x[None] if x.ndim == 2 else x for x in (q, k, v))
        if not (q.shape[0] == k.shape[0] == v.shape[0]):
            raise TensorFileError(f"{cfg.k_path}: heads {k.shape[0]} / {cfg.v_path}: {v.shape[0]} "
                                  f"differ from {cfg.q_path}: {q.shape[0]}")
        if q.shape[2] != k.shape[2]:
            raise TensorFileError(f"{cfg.k_path}: head dim {k.shape[2]} != {cfg.q_path}: {q.shape[2]}")
        if k.shape[1] != v.shape[1]:
            raise TensorFileError(f"{cfg.v_path}: length {v.shape[1]} != {cfg.k_path}: {k.shape[1]}")
        if cfg.causal and q.shape[1] != k.shape[1]:
            raise TensorFileError(f"{cfg.q_path}: causal attention needs len_q == len_k "
                                  f"({q.shape[1]} vs {k.shape[1]})")
        return q, k, v
    return generate_tensors(cfg.seq_len, cfg.seq_len_k or cfg.seq_len, cfg.head_dim, cfg.heads, cfg.seed,
                            cfg.stddev)


# ---------------------------------------------------------------- experiment
def run_experiment(cfg: RunConfig) -> list[dict]:
    """for every sweep point quantize + run DMA on the GPU, compare with the
    full-precision reference (computed once per input head) and return one flat report row
    per (point, head), in sweep order."""
    import torch

    from .attention import dma_attention
    from .metrics import high_precision_fraction, similarity
    from .scores import mixed_precision_scores, reference_attention, reference_scores, score_similarity

    cfg.validate()
    q, k, v = load_inputs(cfg)
    heads, lq, d = q.shape
    lk = k.shape[1]
    qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (q, k, v))
    # score targets above 2^24 cells per head use the row-blocked metric (no N x N matrices)
    tiled = cfg.target == "scores" and lq * lk > (1 << 24)
    if cfg.target == "output":
        refs = [reference_attention(qd[h], kd[h], vd[h], causal=cfg.causal) for h in range(heads)]
    elif not tiled:
        refs = [reference_scores(qd[h], kd[h], causal=cfg.causal) for h in range(heads)]
    rows = []
    for fmt, diag, sink, gran in cfg.points():
        acfg = attention_config(cfg, fmt, diag, sink, gran)
        if cfg.target == "output":
            o = dma_attention(qd[None], kd[None], vd[None], acfg, out_dtype=torch.float32)[0]
            tests = [o[h] for h in range(heads)]
        elif not tiled:
            tests = [mixed_precision_scores(qd[h], kd[h], acfg) for h in range(heads)]
        hp = high_precision_fraction(lq, lk, cfg.tile_m, cfg.tile_n, diag, sink, cfg.causal)
        for h in range(heads):
            m = score_similarity(qd[h], kd[h], acfg) if tiled else similarity(refs[h], tests[h])
            rows.append({
                "cos_sim": m.cos_sim, "rel_l1": m.rel_l1, "abs_l1": m.abs_l1, "rmse": m.rmse, "psnr": m.psnr,
                "high_precision_pct": 100.0 * hp, "seed": None if cfg.q_path else cfg.seed,
                "target": cfg.target, "format": fmt, "diag_window": diag, "sink_window": sink,
                "granularity": gran, "causal": cfg.causal, "tile_m": cfg.tile_m, "tile_n": cfg.tile_n,
                "pv_mode": cfg.pv_mode, "head": h, "len_q": lq, "len_k": lk, "head_dim": d,
            })
    return rows


def format_report(rows: list[dict], kind: str = "json") -> str:
    """JSON: one top-level array of flat objects; CSV: header + one line per row.
    Floats use repr, so identical rows give byte-identical reports."""
    if kind == "json":
        return json.dumps(rows, indent=1, allow_nan=True) + "\n"
    buf = io.StringIO()
    if rows:
        w = csv.DictWriter(buf, fieldnames=list(rows[0]), lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
    return buf.getvalue()


def parse_args(argv=None) -> RunConfig:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_03950_b200.harness",
                                 description="DMA precision sweeps (SPEC.md harness_cli)")
    ap.add_argument("--seq-len", type=int, default=1024)
    ap.add_argument("--seq-len-k", type=int, default=None)
    ap.add_argument("--head-dim", type=int, default=64)
    ap.add_argument("--heads", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--stddev", type=float, default=1.0)
    ap.add_argument("--format", nargs="+", default=["nvfp4"], choices=FORMAT_NAMES)
    ap.add_argument("--diag", nargs="+", type=int, default=[128])
    ap.add_argument("--sink", nargs="+", type=int, default=[128])
    ap.add_argument("--granularity", nargs="+", default=["token"], choices=GRANULARITY_NAMES)
    ap.add_argument("--causal", dest="causal", action="store_true", default=True)
    ap.add_argument("--non-causal", dest="causal", action="store_false")
    ap.add_argument("--tile-m", type=int, default=128)
    ap.add_argument("--tile-n", type=int, default=128)
    ap.add_argument("--pv-mode", default="mxfp8", choices=["mxfp8", "bf16"])
    ap.add_argument("--target", default="output", choices=["output", "scores"])
    ap.add_argument("--q")
    ap.add_argument("--k")
    ap.add_argument("--v")
    ap.add_argument("--out")
    ap.add_argument("--report", default="json", choices=["json", "csv"])
    a = ap.parse_args(argv)
    cfg = RunConfig(seq_len=a.seq_len, seq_len_k=a.seq_len_k, head_dim=a.head_dim, heads=a.heads, seed=a.seed,
                    stddev=a.stddev, q_path=a.q, k_path=a.k, v_path=a.v, formats=a.format, diag=a.diag,
                    sink=a.sink, granularity=a.granularity, causal=a.causal, tile_m=a.tile_m, tile_n=a.tile_n,
                    pv_mode=a.pv_mode, target=a.target, out=a.out, report=a.report)
    cfg.validate()
    return cfg


def main(argv=None) -> int:
    cfg = parse_args(argv)
    text = format_report(run_experiment(cfg), cfg.report)
    if cfg.out:
        with open(cfg.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
