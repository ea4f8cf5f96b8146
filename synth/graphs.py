"""Seeded synthetic FT workloads (graphs + int64 cost tables).

This module is the ONLY code shared by the oracle side (``oracle/``, tests) and
the CUDA side (``paper_2004_10856_b200``, bench).  It holds none of the
method's arithmetic: it only draws graphs and Eq. 1 / Eq. 2 cost tables.

Citations: ``P:n`` = /root/reference/PAPER.md line n (read at build time only,
never at run time); recipe = SURVEY.md §8(d) "Synthetic inputs".

* Operator cost (Eq. 1): ``m = m_p + m_t`` bytes, ``t = t_c + t_s`` ns.
* Edge cost (Eq. 2): ``m = 0``, ``t = t_x`` ns.
* Costs are int64 (reading R10); every value is in [0, 2**40).

Workloads (BASELINE.json ``configs``):

* C1  4-op chain, K=3, integer costs U{0..100}            (brute-forceable)
* C2  VGG-16 chain, D=8 devices  -> K=16
* C3  ResNet-50 with residual branches, D=16 -> K=25
* C4  BERT-large encoder, D=32 -> K=36 (attention mask: K=1 source)
* C5  random two-terminal series-parallel DAG, 2,000 ops, K=64
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np

COST_LIMIT = 1 << 40  # DESIGN.md R10: every input cost in [0, 2^40)


@dataclasses.dataclass
class Workload:
    name: str
    n_cfgs: np.ndarray              # int32[n_ops]  K_i
    src: np.ndarray                 # int32[n_edges]
    dst: np.ndarray                 # int32[n_edges]
    op_m: List[np.ndarray]          # int64[K_i] per op
    op_t: List[np.ndarray]          # int64[K_i] per op
    edge_t: List[np.ndarray]        # int64[K_src*K_dst] row-major [s_src][s_dst]
    edge_m: Optional[List[np.ndarray]] = None  # None -> all zero (Eq. 2)
    op_names: Optional[List[str]] = None
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n_ops(self) -> int:
        return int(len(self.n_cfgs))

    @property
    def n_edges(self) -> int:
        return int(len(self.src))

    def check(self) -> "Workload":
        n = self.n_ops
        assert len(self.op_m) == n and len(self.op_t) == n
        assert len(self.dst) == len(self.src) == len(self.edge_t)
        for i in range(n):
            k = int(self.n_cfgs[i])
            assert k >= 1
            for a in (self.op_m[i], self.op_t[i]):
                assert a.dtype == np.int64 and a.shape == (k,)
                assert a.min() >= 0 and a.max() < COST_LIMIT
        for e in range(self.n_edges):
            s, d = int(self.src[e]), int(self.dst[e])
            assert 0 <= s < n and 0 <= d < n and s != d
            shape = (int(self.n_cfgs[s]) * int(self.n_cfgs[d]),)
            arrs = [self.edge_t[e]] + ([self.edge_m[e]] if self.edge_m is not None else [])
            for a in arrs:
                assert a.dtype == np.int64 and a.shape == shape, (e, a.shape, shape)
                assert a.min() >= 0 and a.max() < COST_LIMIT
        return self


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


# --------------------------------------------------------------------------
# C1 and tiny random fixtures (brute-force checkable)
# --------------------------------------------------------------------------

def random_graph(n_ops: int, edges: List[Tuple[int, int]], K, seed: int,
                 cost_hi: int = 100, edge_mem: bool = False, name: str = "random") -> Workload:
    """Integer costs U{0..cost_hi} drawn in the SURVEY §8(d) C1 order:
    ops by id (m then t), then edges by id (t, then m if ``edge_mem``)."""
    rng = np.random.default_rng(seed)
    if isinstance(K, int):
        K = [K] * n_ops
    K = np.asarray(K, dtype=np.int32)
    op_m, op_t = [], []
    for i in range(n_ops):
        op_m.append(_i64(rng.integers(0, cost_hi + 1, int(K[i]))))
        op_t.append(_i64(rng.integers(0, cost_hi + 1, int(K[i]))))
    edge_t, edge_m = [], []
    for (s, d) in edges:
        edge_t.append(_i64(rng.integers(0, cost_hi + 1, (int(K[s]) * int(K[d]),))))
        if edge_mem:
            edge_m.append(_i64(rng.integers(0, cost_hi + 1, (int(K[s]) * int(K[d]),))))
    src = np.asarray([e[0] for e in edges], dtype=np.int32)
    dst = np.asarray([e[1] for e in edges], dtype=np.int32)
    return Workload(name, K, src, dst, op_m, op_t, edge_t,
                    edge_m if edge_mem else None).check()


def c1(seed: int = 0, variant: str = "chain") -> Workload:
    """C1: 4-op chain o0->o1->o2->o3, K=3, m,t ~ U{0..100}, edge t ~ U{0..100}.
    Variants: ``chain``; ``parallel`` (+1 parallel edge o1->o2); ``diamond``
    (o0->o1, o0->o2, o1->o3, o2->o3)."""
    if variant == "chain":
        edges = [(0, 1), (1, 2), (2, 3)]
    elif variant == "parallel":
        edges = [(0, 1), (1, 2), (2, 3), (1, 2)]
    elif variant == "diamond":
        edges = [(0, 1), (0, 2), (1, 3), (2, 3)]
    else:
        raise ValueError(variant)
    return random_graph(4, edges, 3, seed, name=f"C1-{variant}-s{seed}")


# --------------------------------------------------------------------------
# C2-C4: DNN graphs with the SURVEY §8(d) common cost model
# --------------------------------------------------------------------------

N_BATCH = 256          # T-model batch size
FP32_NS = 15.7e3       # flops per ns (V100 fp32, 15.7 TFLOP/s)


def config_space(D: int) -> List[Tuple[int, int, int]]:
    """(b, h, v): batch split b, model split h (powers of 2, b*h | D),
    variant v in {0,1} when h > 1.  Sorted by (b*h, b, v).  K(8)=16,
    K(16)=25, K(32)=36.  Stands in for the withheld enumeration rules."""
    out = []
    p = 1
    pw = []
    while p <= D:
        pw.append(p)
        p *= 2
    for b in pw:
        for h in pw:
            if b * h > D or D % (b * h):
                continue
            for v in ((0, 1) if h > 1 else (0,)):
                out.append((b, h, v))
    out.sort(key=lambda c: (c[0] * c[1], c[0], c[2]))
    return out


def _beta(g: int) -> float:
    """Bytes per ns: NVLink inside a machine (g <= 8), EDR IB across."""
    return 100.0 if g <= 8 else 12.5


@dataclasses.dataclass
class OpSpec:
    name: str
    P: float  # parameter bytes
    A: float  # activation bytes
    F: float  # flops (fwd+bwd)


def _op_costs(spec: OpSpec, cfgs, D: int) -> Tuple[np.ndarray, np.ndarray]:
    m = np.empty(len(cfgs))
    t = np.empty(len(cfgs))
    for c, (b, h, v) in enumerate(cfgs):
        m[c] = spec.P / h + spec.A / (b * h)
        tc = math.floor(spec.F / (b * h) / FP32_NS)
        g = D // h
        if spec.P > 0 and g > 1:
            ts = 10_000.0 + 2.0 * (g - 1) / g * (spec.P / h) / _beta(g)
        else:
            ts = 0.0
        t[c] = tc + ts
    return m, t


def _edge_cost(a_src: float, cfgs_s, cfgs_d, D: int) -> np.ndarray:
    ks, kd = len(cfgs_s), len(cfgs_d)
    out = np.zeros((ks, kd), dtype=np.int64)
    beta = _beta(D)
    for i, (b, h, v) in enumerate(cfgs_s):
        for j, (b2, h2, v2) in enumerate(cfgs_d):
            if (b, h, v) == (b2, h2, v2):
                continue
            out[i, j] = math.floor(10_000.0 + (a_src / min(b * h, b2 * h2)) / beta)
    return out.reshape(-1)


def _dnn_workload(name: str, specs: List[OpSpec], edges: List[Tuple[int, int]], D: int,
                  seed: int = 0, jitter: bool = True, k1_ops=(), const_edge_t=None) -> Workload:
    """Build a workload from op specs.  ``k1_ops``: ops with a single config
    (replicated); ``const_edge_t``: {edge index: constant t} overrides."""
    cfgs = config_space(D)
    rng = np.random.default_rng(seed)
    n = len(specs)
    K = np.asarray([1 if i in k1_ops else len(cfgs) for i in range(n)], dtype=np.int32)
    op_m, op_t = [], []
    for i, spec in enumerate(specs):
        cf = [(1, 1, 0)] if i in k1_ops else cfgs
        m, t = _op_costs(spec, cf, D)
        if jitter:  # draw order: op by id, cfg in canonical order, m then t
            for c in range(len(cf)):
                m[c] *= 1.0 + rng.random() / 64.0
                t[c] *= 1.0 + rng.random() / 64.0
        op_m.append(_i64(np.floor(m)))
        op_t.append(_i64(np.floor(t)))
    edge_t = []
    const_edge_t = const_edge_t or {}
    for e, (s, d) in enumerate(edges):
        cs = [(1, 1, 0)] if s in k1_ops else cfgs
        cd = [(1, 1, 0)] if d in k1_ops else cfgs
        if e in const_edge_t:
            edge_t.append(_i64(np.full(len(cs) * len(cd), const_edge_t[e])))
        else:
            edge_t.append(_edge_cost(specs[s].A, cs, cd, D))
    src = np.asarray([e[0] for e in edges], dtype=np.int32)
    dst = np.asarray([e[1] for e in edges], dtype=np.int32)
    return Workload(name, K, src, dst, op_m, op_t, edge_t, None,
                    [s.name for s in specs], {"D": D, "K": len(cfgs), "seed": seed,
                                              "jitter": jitter}).check()


def _conv(name, k, cin, cout, H, N=N_BATCH):
    return OpSpec(name, 4.0 * (k * k * cin * cout + cout), 4.0 * N * cout * H * H,
                  6.0 * N * H * H * k * k * cin * cout)


def _fc(name, fin, fout, rows):
    return OpSpec(name, 4.0 * (fin * fout + fout), 4.0 * rows * fout, 6.0 * rows * fin * fout)


def _elt(name, elems, fl_per_elem, P=0.0):
    return OpSpec(name, P, 4.0 * elems, fl_per_elem * elems)


def c2(seed: int = 0, jitter: bool = True) -> Workload:
    """C2: VGG-16 as a 23-op chain (input, 13 conv, 5 pool, 3 FC, loss), D=8."""
    N = N_BATCH
    specs = [OpSpec("input", 0.0, 4.0 * N * 3 * 224 * 224, 0.0)]
    cin, H = 3, 224
    for stage, (width, reps) in enumerate([(64, 2), (128, 2), (256, 3), (512, 3), (512, 3)]):
        for r in range(reps):
            specs.append(_conv(f"conv{stage + 1}_{r + 1}", 3, cin, width, H))
            cin = width
        specs.append(_elt(f"pool{stage + 1}", N * cin * (H // 2) ** 2, 3.0 * 4))
        H //= 2
    specs.append(_fc("fc6", 512 * 7 * 7, 4096, N))
    specs.append(_fc("fc7", 4096, 4096, N))
    specs.append(_fc("fc8", 4096, 1000, N))
    specs.append(OpSpec("loss", 0.0, 4.0 * N, 6.0 * N * 1000))
    edges = [(i, i + 1) for i in range(len(specs) - 1)]
    assert len(specs) == 23 and len(edges) == 22
    return _dnn_workload("C2-vgg16", specs, edges, 8, seed, jitter)


def c3(seed: int = 0, jitter: bool = True) -> Workload:
    """C3: ResNet-50 (74 ops / 89 edges) with residual branches, D=16."""
    N = N_BATCH
    specs: List[OpSpec] = []
    edges: List[Tuple[int, int]] = []

    def add(spec):
        specs.append(spec)
        return len(specs) - 1

    x = add(OpSpec("input", 0.0, 4.0 * N * 3 * 224 * 224, 0.0))
    c = add(_conv("conv1", 7, 3, 64, 112))
    edges.append((x, c))
    p = add(_elt("maxpool", N * 64 * 56 * 56, 3.0 * 4))
    edges.append((c, p))
    prev, cin, H = p, 64, 56
    for stage, (w, reps) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        for r in range(reps):
            Hout = H // 2 if (r == 0 and stage > 0) else H
            a = add(_conv(f"s{stage}b{r}a", 1, cin, w, H))
            edges.append((prev, a))
            bb = add(_conv(f"s{stage}b{r}b", 3, w, w, Hout))
            edges.append((a, bb))
            cc = add(_conv(f"s{stage}b{r}c", 1, w, 4 * w, Hout))
            edges.append((bb, cc))
            s = add(_elt(f"s{stage}b{r}add", N * 4 * w * Hout * Hout, 3.0))
            edges.append((cc, s))
            if r == 0:
                pr = add(_conv(f"s{stage}proj", 1, cin, 4 * w, Hout))
                edges.append((prev, pr))
                edges.append((pr, s))
            else:
                edges.append((prev, s))
            prev, cin, H = s, 4 * w, Hout
    ap = add(_elt("avgpool", N * 2048, 3.0 * 49))
    edges.append((prev, ap))
    fc = add(_fc("fc", 2048, 1000, N))
    edges.append((ap, fc))
    ls = add(OpSpec("loss", 0.0, 4.0 * N, 6.0 * N * 1000))
    edges.append((fc, ls))
    assert len(specs) == 74 and len(edges) == 89, (len(specs), len(edges))
    return _dnn_workload("C3-resnet50", specs, edges, 16, seed, jitter)


def c4(seed: int = 0, jitter: bool = True, layers: int = 24, mask_k1: bool = True) -> Workload:
    """C4: BERT-large encoder (342 ops / 460 edges at 24 layers), D=32.
    The attention mask is a K=1 source feeding every scores op;
    mask edges carry t = 10,000 ns.  mask_k1=False gives the mask the full
    configuration space (the case heuristic elimination, Eq. 7, exists for)."""
    N, S, H, heads = N_BATCH, 128, 1024, 16
    rows = N * S
    specs: List[OpSpec] = []
    edges: List[Tuple[int, int]] = []
    const_t = {}

    def add(spec):
        specs.append(spec)
        return len(specs) - 1

    ids = add(OpSpec("ids", 0.0, 4.0 * N * S, 0.0))
    mask = add(OpSpec("mask", 0.0, 4.0 * N * S, 0.0))
    emb = add(OpSpec("embedding", 4.0 * (30522 + 512 + 2) * H, 4.0 * rows * H, 6.0 * rows * H))
    edges.append((ids, emb))
    prev = emb
    for L in range(layers):
        q = add(_fc(f"L{L}q", H, H, rows))
        k = add(_fc(f"L{L}k", H, H, rows))
        v = add(_fc(f"L{L}v", H, H, rows))
        sc = add(OpSpec(f"L{L}scores", 0.0, 4.0 * N * heads * S * S, 6.0 * N * S * S * H))
        sm = add(_elt(f"L{L}softmax", N * heads * S * S, 8.0))
        av = add(OpSpec(f"L{L}attnv", 0.0, 4.0 * rows * H, 6.0 * N * S * S * H))
        o = add(_fc(f"L{L}out", H, H, rows))
        a1 = add(_elt(f"L{L}add1", rows * H, 3.0))
        n1 = add(_elt(f"L{L}ln1", rows * H, 8.0, P=8.0 * H))
        f1 = add(_fc(f"L{L}ffn1", H, 4 * H, rows))
        ge = add(_elt(f"L{L}gelu", rows * 4 * H, 8.0))
        f2 = add(_fc(f"L{L}ffn2", 4 * H, H, rows))
        a2 = add(_elt(f"L{L}add2", rows * H, 3.0))
        n2 = add(_elt(f"L{L}ln2", rows * H, 8.0, P=8.0 * H))
        for (s_, d_) in [(prev, q), (prev, k), (prev, v), (q, sc), (k, sc)]:
            edges.append((s_, d_))
        const_t[len(edges)] = 10_000
        edges.append((mask, sc))
        for (s_, d_) in [(sc, sm), (sm, av), (v, av), (av, o), (o, a1), (prev, a1), (a1, n1),
                         (n1, f1), (f1, ge), (ge, f2), (f2, a2), (n1, a2), (a2, n2)]:
            edges.append((s_, d_))
        prev = n2
    po = add(_fc("pooler", H, H, N))
    edges.append((prev, po))
    cl = add(_fc("classifier", H, 2, N))
    edges.append((po, cl))
    ls = add(OpSpec("loss", 0.0, 4.0 * N, 6.0 * N * 2))
    edges.append((cl, ls))
    if layers == 24:
        assert len(specs) == 342 and len(edges) == 460, (len(specs), len(edges))
    return _dnn_workload(f"C4-bert-large-L{layers}", specs, edges, 32, seed, jitter,
                         k1_ops=(mask,) if mask_k1 else (), const_edge_t=const_t)


# --------------------------------------------------------------------------
# C5: random two-terminal series-parallel DAG
# --------------------------------------------------------------------------

def c5(seed: int = 0, n_ops: int = 2000, K: int = 64, B: int = 32, Lmin: int = 4,
       Lmax: int = 8, rho: float = 0.99) -> Workload:
    """C5 (SURVEY §8(d) pseudo-code): backbone of B ops, parallel chains of
    U{Lmin..Lmax} ops added round-robin over the spans, U{1..3} per visit,
    until ``n_ops`` ops.  Op m = floor(2^24 u), t = floor(2^24 (rho u + (1-rho) w));
    edge t = 0 w.p. 1/4, else floor(2^24 (1-rho) U[0,1)).

    Calibrated defaults (SURVEY 8(d) "C5 calibration", measured on B200 with
    libft): rho = 0.99, B = 32, L in {4..8} give 2.70e10
    product tuples, max segment frontier 21,598, final frontier 16,912.
    The survey's starting point (rho = 0.85, L in {4..12}) gives 6.2e12."""
    rng = np.random.default_rng(seed)
    edges: List[Tuple[int, int]] = [(s, s + 1) for s in range(B - 1)]
    n = B
    s = 0
    done = n >= n_ops
    while not done:
        for _ in range(int(rng.integers(1, 4))):
            L = min(int(rng.integers(Lmin, Lmax + 1)), n_ops - n)
            if L == 0:
                done = True
                break
            chain = list(range(n, n + L))
            n += L
            edges.append((s, chain[0]))
            for a, b in zip(chain[:-1], chain[1:]):
                edges.append((a, b))
            edges.append((chain[-1], s + 1))
            if n >= n_ops:
                done = True
                break
        s = (s + 1) % (B - 1)
    Ks = np.full(n, K, dtype=np.int32)
    op_m, op_t = [], []
    scale = float(1 << 24)
    for _ in range(n):
        u = rng.random(K)
        w = rng.random(K)
        op_m.append(_i64(np.floor(scale * u)))
        op_t.append(_i64(np.floor(scale * (rho * u + (1.0 - rho) * w))))
    edge_t = []
    for _ in edges:
        z = rng.random((K, K)) < 0.25
        tt = np.floor(scale * (1.0 - rho) * rng.random((K, K)))
        edge_t.append(_i64(np.where(z, 0.0, tt).reshape(-1)))
    src = np.asarray([e[0] for e in edges], dtype=np.int32)
    dst = np.asarray([e[1] for e in edges], dtype=np.int32)
    return Workload(f"C5-spdag-n{n}-K{K}", Ks, src, dst, op_m, op_t, edge_t, None, None,
                    {"B": B, "Lmin": Lmin, "Lmax": Lmax, "rho": rho, "seed": seed}).check()


def big_chain(seed: int = 0, n_ops: int = 16384, K: int = 2, rho: float = 0.95,
              span: int = 1 << 16) -> Workload:
    """Wide-cost chain (R10 range test): o_0 -> ... -> o_{n-1}, K configs.
    Every op and edge cost has m = 2^40 - 1 - span + floor(span u) (edge
    memory included, R11) and t = floor(span (rho u + (1 - rho) w)), u, w ~
    U[0,1) per entry: each input cost sits just below the 2^40 bound, so the
    frontier m of an i-op prefix is about i 2^40 (2^55 at 16,384 ops) while
    its spread stays small; rho keeps the frontiers bounded (as in C5).
    Draw order: ops (u, w) by id, then edges (u, w) by id."""
    rng = np.random.default_rng(seed)
    base = float((1 << 40) - 1 - span)
    op_m, op_t = [], []
    for _ in range(n_ops):
        u = rng.random(K)
        w = rng.random(K)
        op_m.append(_i64(base + np.floor(span * u)))
        op_t.append(_i64(np.floor(span * (rho * u + (1.0 - rho) * w))))
    edge_m, edge_t = [], []
    for _ in range(n_ops - 1):
        u = rng.random(K * K)
        w = rng.random(K * K)
        edge_m.append(_i64(base + np.floor(span * u)))
        edge_t.append(_i64(np.floor(span * (rho * u + (1.0 - rho) * w))))
    src = np.arange(n_ops - 1, dtype=np.int32)
    return Workload(f"bigchain-n{n_ops}-K{K}", np.full(n_ops, K, np.int32), src, src + 1, op_m, op_t,
                    edge_t, edge_m, None, {"rho": rho, "span": span, "seed": seed}).check()


def scaled(w: Workload, bits: int = 40) -> Workload:
    """The same graph with every cost multiplied by one integer factor so
    that the largest cost is just below 2^bits (R10's bound at bits = 40)."""
    mx = max([int(a.max()) for a in w.op_m + w.op_t + w.edge_t] +
             [int(a.max()) for a in (w.edge_m or [])] + [1])
    f = ((1 << bits) - 1) // mx
    mul = lambda L: None if L is None else [_i64(a * f) for a in L]
    return Workload(w.name + f"-x{f}", w.n_cfgs, w.src, w.dst, mul(w.op_m), mul(w.op_t),
                    mul(w.edge_t), mul(w.edge_m), w.op_names, dict(w.meta, scale=f)).check()


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def get(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)


def random_leafy(seed: int, n_ops: int = 5, kmax: int = 3, leaves: int = 2, cost_hi: int = 8,
                 edge_mem: bool = False) -> Workload:
    """A random SP graph with `leaves` extra ops attached by a single edge
    (an input feeding, or an output read from, a random op) -- shapes that
    need branch elimination (Eq. 6).  Costs U{0..cost_hi}, seeded."""
    base = random_sp(seed, n_ops=n_ops, kmax=kmax, p_mask=0.0, cost_hi=cost_hi, edge_mem=edge_mem)
    rng = np.random.default_rng(seed + 7919)
    K = [int(k) for k in base.n_cfgs]
    edges = list(zip(base.src.tolist(), base.dst.tolist()))
    has_in = {d for _, d in edges}
    has_out = {a for a, _ in edges}
    for _ in range(leaves):
        # an input leaf goes to an op that already has an input, an output leaf
        # to one that already has an output (the graph's source stays the
        # backbone head), both to ops with K >= 2 (a K=1 source with an
        # extra output would be folded first, Eq. 7, disconnecting its consumers)
        as_input = rng.integers(0, 2) == 0
        cand = [v for v in range(len(K)) if K[v] >= 2 and (v in has_in if as_input else v in has_out)]
        if not cand:
            continue
        h = int(cand[int(rng.integers(0, len(cand)))])
        i = len(K)
        K.append(int(rng.integers(2, max(2, kmax) + 1)))
        edges.append((i, h) if as_input else (h, i))
    w = random_graph(len(K), edges, K, seed + 104729, cost_hi=cost_hi, edge_mem=edge_mem,
                     name=f"leafy{seed}")
    return w


def random_masked(seed: int, n_ops: int = 5, kmax: int = 3, mask_k: int = 2, fanout: int = 2,
                  cost_hi: int = 8) -> Workload:
    """A random SP graph plus a BERT-mask-like source (the last op id, so
    not the backbone head) with `mask_k` >= 2 configurations feeding
    `fanout` random non-source ops -- the shape heuristic elimination (Eq. 7)
    is for.  Costs U{0..cost_hi}, seeded."""
    base = random_sp(seed, n_ops=n_ops, kmax=kmax, p_mask=0.0, cost_hi=cost_hi)
    rng = np.random.default_rng(seed + 15485863)
    K = [int(k) for k in base.n_cfgs] + [int(mask_k)]
    edges = list(zip(base.src.tolist(), base.dst.tolist()))
    targets = sorted({d for _, d in edges})
    m = len(K) - 1
    for d in rng.choice(targets, size=min(fanout, len(targets)), replace=False).tolist():
        edges.append((m, int(d)))
    return random_graph(len(K), edges, K, seed + 32452843, cost_hi=cost_hi, name=f"masked{seed}")


def random_dag(seed: int, n_ops: int = 6, kmax: int = 3, p_edge: float = 0.4, cost_hi: int = 8,
               edge_mem: bool = False) -> Workload:
    """Small random DAG, in general NOT series-parallel (brute-force fixtures
    for composite branch elimination, Eq. 6): ops 0..n-1 in topological id
    order; every op v > 0 gets an input from a random u < v, every op
    v < n-1 an output to a random later op, and every other pair u < v an
    edge with probability ``p_edge``.  K ~ U{1..kmax}; costs U{0..cost_hi}."""
    rng = np.random.default_rng(seed)
    E = set()
    for v in range(1, n_ops):
        E.add((int(rng.integers(0, v)), v))
    for u in range(n_ops - 1):
        E.add((u, int(rng.integers(u + 1, n_ops))))
    for u in range(n_ops):
        for v in range(u + 1, n_ops):
            if rng.random() < p_edge:
                E.add((u, v))
    K = [int(rng.integers(1, kmax + 1)) for _ in range(n_ops)]
    return random_graph(n_ops, sorted(E), K, seed + 7919, cost_hi=cost_hi, edge_mem=edge_mem,
                        name=f"dag-s{seed}")


def random_sp(seed: int, n_ops: int = 6, kmax: int = 3, p_parallel: float = 0.35,
              p_mask: float = 0.3, cost_hi: int = 8, edge_mem: bool = False) -> Workload:
    """Small random two-terminal series-parallel DAG (brute-force fixtures).

    Built from one edge 0->1 by random series splits (u->v => u->x->v) and
    parallel additions (a second edge u->v or a parallel 1-op chain), plus,
    with probability ``p_mask``, a K=1 source feeding 1..3 non-source ops (the
    BERT-mask structure of P:618).  Small cost range -> many exact ties."""
    rng = np.random.default_rng(seed)
    edges: List[Tuple[int, int]] = [(0, 1)]
    n = 2
    mask_budget = 1 if rng.random() < p_mask else 0
    while n < n_ops - mask_budget:
        e = int(rng.integers(0, len(edges)))
        u, v = edges[e]
        r = rng.random()
        if r < p_parallel:
            if rng.random() < 0.5:
                edges.append((u, v))
            else:
                edges.append((u, n))
                edges.append((n, v))
                n += 1
        else:
            edges[e] = (u, n)
            edges.append((n, v))
            n += 1
    K = [int(rng.integers(1, kmax + 1)) for _ in range(n)]
    if mask_budget:
        mk = n
        n += 1
        K.append(1)
        targets = rng.choice(np.arange(1, n - 1), size=min(n - 2, int(rng.integers(1, 4))),
                             replace=False)
        for tg in sorted(int(x) for x in targets):
            edges.append((mk, tg))
    return random_graph(n, edges, K, seed + 7919, cost_hi=cost_hi, edge_mem=edge_mem,
                        name=f"spdag-s{seed}")
