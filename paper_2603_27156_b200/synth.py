"""Synthetic circuit-like graphs — host-side input producer.

Restates SPEC `generate_synthetic` and
`from_edge_list`: a near-regular ring lattice of
`base_degree` plus `hub_fraction·n` star hubs whose degrees are drawn from
`hub_degree_range` (uniform, or a power law for the 10M-node depth-stress
config), symmetrised ("default to symmetrized input"),
deduplicated and row-sorted. Labels are a degree-weighted congestion proxy
smoothed over `label_smoothing_hops`, min-max scaled to [0, 1] plus Gaussian
noise; features are degree, local clustering and random channels; masks split
80/10/10 by seeded shuffle (0=train, 1=val, 2=test).

Seeded-deterministic (numpy PCG64); vectorised so 10M-node graphs build in
seconds. This is not on the device hot path; it produces the CSR that the
C-ABI uploads (`gsrc_graph_upload`).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SynthConfig:
    """SynthConfig."""

    n: int = 10_000
    base_degree: int = 2
    hub_fraction: float = 0.002
    hub_degree_range: tuple = (300, 700)
    label_smoothing_hops: int = 2
    noise_std: float = 0.02
    seed: int = 0
    d_in: int = 8
    power_law: bool = False      # hub degrees ~ Pareto(1.5) clipped to the range
    self_loops: bool = False

    def validate(self):
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if not 0.0 <= self.hub_fraction <= 1.0:
            raise ValueError("hub_fraction must be in [0,1]")
        lo, hi = self.hub_degree_range
        if self.hub_fraction > 0 and not (0 < lo <= hi < self.n):
            raise ValueError(f"infeasible hub_degree_range {self.hub_degree_range} for n={self.n}")
        if self.base_degree < 0 or self.base_degree >= self.n:
            raise ValueError("infeasible base_degree")
        if self.d_in < 2:
            raise ValueError("d_in must be >= 2 (degree, clustering, random...)")


@dataclass
class CsrGraph:
    """CsrGraph: int64 row_ptr, int32 col_idx (ascending, unique)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray

    @property
    def e(self):
        return int(self.col_idx.size)

    def degree(self):
        return np.diff(self.row_ptr)


@dataclass
class NodeData:
    """NodeData."""

    features: np.ndarray   # n × d_in float32
    labels: np.ndarray     # n float32
    split: np.ndarray      # n uint8: 0 train, 1 val, 2 test

    @property
    def train_mask(self):
        return (self.split == 0).astype(np.uint8)


def from_edge_list(n: int, u: np.ndarray, v: np.ndarray) -> CsrGraph:
    """Deduplicated, row-sorted CSR."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    if u.size and (u.min() < 0 or v.min() < 0 or u.max() >= n or v.max() >= n):
        raise ValueError("edge endpoint out of range")
    codes = np.unique(u * n + v)
    rows = codes // n
    cols = (codes % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return CsrGraph(n=n, row_ptr=row_ptr, col_idx=cols)


def _hub_edges(cfg: SynthConfig, rng: np.random.Generator):
    n = cfg.n
    nh = int(round(cfg.hub_fraction * n))
    if nh == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    hubs = rng.choice(n, size=nh, replace=False)
    lo, hi = cfg.hub_degree_range
    if cfg.power_law:
        deg = lo * (1.0 + rng.pareto(1.5, size=nh))
        deg = np.clip(deg, lo, hi).astype(np.int64)
    else:
        deg = rng.integers(lo, hi + 1, size=nh)
    src = np.repeat(hubs.astype(np.int64), deg)
    dst = rng.integers(0, n, size=int(deg.sum()), dtype=np.int64)
    keep = src != dst
    return src[keep], dst[keep]


def generate_graph(cfg: SynthConfig) -> CsrGraph:
    cfg.validate()
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    n = cfg.n
    base = np.arange(n, dtype=np.int64)
    us, vs = [], []
    for off in range(1, cfg.base_degree // 2 + 1):
        us.append(base)
        vs.append((base + off) % n)
    if cfg.base_degree % 2:  # odd base degree: add a chord to the node n/2 away
        us.append(base)
        vs.append((base + n // 2) % n)
    hu, hv = _hub_edges(cfg, rng)
    us.append(hu)
    vs.append(hv)
    u = np.concatenate(us)
    v = np.concatenate(vs)
    keep = u != v
    u, v = u[keep], v[keep]
    uu = np.concatenate([u, v])
    vv = np.concatenate([v, u])
    if cfg.self_loops:
        uu = np.concatenate([uu, base])
        vv = np.concatenate([vv, base])
    return from_edge_list(n, uu, vv)


def _row_mean(g: CsrGraph, x: np.ndarray) -> np.ndarray:
    deg = g.degree()
    rows = np.repeat(np.arange(g.n), deg)
    s = np.bincount(rows, weights=x[g.col_idx], minlength=g.n)
    return np.where(deg > 0, s / np.maximum(deg, 1), 0.0)


def _clustering(g: CsrGraph, max_deg: int = 64) -> np.ndarray:
    """Local clustering coefficient on the subgraph of nodes with degree <=
    max_deg (hubs excluded, their coefficient reported as 0): exact triangle
    counts without the O(hub_degree²) blow-up."""
    import scipy.sparse as sp

    deg = g.degree()
    small = deg <= max_deg
    rows = np.repeat(np.arange(g.n), deg)
    keep = small[rows] & small[g.col_idx]
    A = sp.csr_matrix((np.ones(int(keep.sum()), np.float64), (rows[keep], g.col_idx[keep])), shape=(g.n, g.n))
    tri = np.asarray((A @ A).multiply(A).sum(axis=1)).ravel() / 2.0
    ds = np.asarray(A.sum(axis=1)).ravel()
    denom = ds * (ds - 1) / 2.0
    return np.where(denom > 0, tri / np.maximum(denom, 1), 0.0)


def generate_node_data(cfg: SynthConfig, g: CsrGraph) -> NodeData:
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 0x9E3779B9))
    n = g.n
    deg = g.degree().astype(np.float64)
    # degree-weighted congestion proxy, smoothed over k hops
    c = np.log1p(deg)
    for _ in range(cfg.label_smoothing_hops):
        c = 0.5 * c + 0.5 * _row_mean(g, c)
    lo, hi = c.min(), c.max()
    lab = (c - lo) / (hi - lo) if hi > lo else np.zeros_like(c)
    lab = lab + rng.normal(0.0, cfg.noise_std, size=n)
    feats = np.empty((n, cfg.d_in), np.float64)
    feats[:, 0] = np.log1p(deg)
    feats[:, 1] = _clustering(g)
    if cfg.d_in > 2:
        feats[:, 2:] = rng.normal(0.0, 1.0, size=(n, cfg.d_in - 2))
    perm = rng.permutation(n)
    split = np.zeros(n, np.uint8)
    n_tr = int(0.8 * n)
    n_va = int(0.1 * n)
    split[perm[n_tr:n_tr + n_va]] = 1
    split[perm[n_tr + n_va:]] = 2
    return NodeData(features=feats.astype(np.float32), labels=lab.astype(np.float32), split=split)


def generate_synthetic(cfg: SynthConfig):
    """(CsrGraph, NodeData) — SPEC.md:186-194."""
    g = generate_graph(cfg)
    return g, generate_node_data(cfg, g)


# Named configurations from BASELINE.json `configs`.
def config_graph(name: str, seed: int = 0) -> SynthConfig:
    name = name.lower()
    if name == "c1":
        return SynthConfig(n=10_000, base_degree=2, hub_fraction=0.002, hub_degree_range=(300, 700), seed=seed)
    if name == "c2":
        return SynthConfig(n=100_000, base_degree=2, hub_fraction=0.002, hub_degree_range=(300, 700), seed=seed)
    if name in ("c3", "c4"):
        return SynthConfig(n=1_000_000, base_degree=2, hub_fraction=0.002, hub_degree_range=(300, 700), seed=seed)
    if name == "c5":
        return SynthConfig(n=10_000_000, base_degree=2, hub_fraction=0.0005, hub_degree_range=(500, 20_000),
                           power_law=True, seed=seed)
    raise ValueError(f"unknown config {name}")


# ---- graph-store binary formats ------------------------------
# GSRG: magic "GSRG", u32 LE version, u64 LE n, u64 LE e, row_ptr (n+1) × i64 LE,
#       col_idx e × i32 LE.
# GSRN: magic "GSRN", u64 LE n, u64 LE d_in, features n×d_in f64 LE (row-major),
#       labels n × f64 LE, split n × u8 (0 train, 1 val, 2 test).
GSRG_VERSION = 1


def write_graph(path: str, g: CsrGraph) -> None:
    with open(path, "wb") as f:
        f.write(b"GSRG")
        f.write(np.array([GSRG_VERSION], "<u4").tobytes())
        f.write(np.array([g.n, g.e], "<u8").tobytes())
        f.write(np.ascontiguousarray(g.row_ptr, "<i8").tobytes())
        f.write(np.ascontiguousarray(g.col_idx, "<i4").tobytes())


def read_graph(path: str) -> CsrGraph:
    """Raises ValueError (FormatError) on bad magic, version, truncation or a malformed CSR."""
    with open(path, "rb") as f:
        buf = f.read()
    if len(buf) < 24 or buf[:4] != b"GSRG":
        raise ValueError(f"{path}: bad GSRG magic")
    ver = int(np.frombuffer(buf, "<u4", 1, 4)[0])
    if ver != GSRG_VERSION:
        raise ValueError(f"{path}: unsupported GSRG version {ver}")
    n, e = (int(x) for x in np.frombuffer(buf, "<u8", 2, 8))
    need = 24 + 8 * (n + 1) + 4 * e
    if len(buf) != need:
        raise ValueError(f"{path}: truncated GSRG ({len(buf)} of {need} bytes)")
    rp = np.frombuffer(buf, "<i8", n + 1, 24).astype(np.int64)
    ci = np.frombuffer(buf, "<i4", e, 24 + 8 * (n + 1)).astype(np.int32)
    if rp[0] != 0 or rp[-1] != e or np.any(np.diff(rp) < 0):
        raise ValueError(f"{path}: malformed row_ptr")
    if e and (ci.min() < 0 or ci.max() >= n):
        raise ValueError(f"{path}: col_idx out of range")
    return CsrGraph(n=n, row_ptr=rp, col_idx=ci)


def write_node_data(path: str, nd: NodeData) -> None:
    n, d_in = nd.features.shape
    with open(path, "wb") as f:
        f.write(b"GSRN")
        f.write(np.array([n, d_in], "<u8").tobytes())
        f.write(np.ascontiguousarray(nd.features, "<f8").tobytes())
        f.write(np.ascontiguousarray(nd.labels, "<f8").tobytes())
        f.write(np.ascontiguousarray(nd.split, np.uint8).tobytes())


def read_node_data(path: str) -> NodeData:
    with open(path, "rb") as f:
        buf = f.read()
    if len(buf) < 20 or buf[:4] != b"GSRN":
        raise ValueError(f"{path}: bad GSRN magic")
    n, d_in = (int(x) for x in np.frombuffer(buf, "<u8", 2, 4))
    need = 20 + 8 * n * d_in + 8 * n + n
    if len(buf) != need:
        raise ValueError(f"{path}: truncated GSRN ({len(buf)} of {need} bytes)")
    feats = np.frombuffer(buf, "<f8", n * d_in, 20).reshape(n, d_in).astype(np.float32)
    labels = np.frombuffer(buf, "<f8", n, 20 + 8 * n * d_in).astype(np.float32)
    split = np.frombuffer(buf, np.uint8, n, 20 + 8 * n * d_in + 8 * n).copy()
    if split.size and split.max() > 2:
        raise ValueError(f"{path}: split code out of range")
    return NodeData(features=feats, labels=labels, split=split)
