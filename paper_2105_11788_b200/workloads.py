"""Synthetic LTS generators for the benchmark configurations (SURVEY §8d,
BASELINE.json `configs`) and an independent ground-truth checker.

Every generator returns int32 columns; none of this is on the refinement
path.  `signature_bisim` is a deliberately different algorithm (iterated
signature refinement) used only to check results where the PRAM oracle
cannot finish.
"""
from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np


@dataclass
class Instance:
    name: str
    kind: str                 # "bcrp" | "rcpp"
    n: int
    src: np.ndarray
    dst: np.ndarray
    act: np.ndarray | None = None
    num_actions: int = 1
    pi0: np.ndarray | None = None   # RCPP leader-form initial partition
    truth: np.ndarray | None = None  # canonical coarsest partition, when known
    expect_supersteps: int | None = None

    @property
    def m(self) -> int:
        return int(self.src.size)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def canonical(assignment: np.ndarray) -> np.ndarray:
    """Leader form with leader = smallest member (lts.py:117-128)."""
    _, first, inv = np.unique(np.asarray(assignment), return_index=True, return_inverse=True)
    return first[inv.reshape(-1)].astype(np.int32)


def c1_random(n: int = 10_000, m: int = 50_000, seed: int = 1) -> Instance:
    """c1: iid (source, label, target), |Act| = 4, drawn exactly as SURVEY §8d
    prescribes with Python's random.Random(seed) so the reference's full run
    (tests/golden/c1_reference.*) applies."""
    rng = random.Random(seed)
    src = np.empty(m, np.int32)
    act = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    rr = rng.randrange
    for i in range(m):
        src[i] = rr(n)
        act[i] = rr(4)   # labels a0..a3 sort to ids 0..3
        dst[i] = rr(n)
    return Instance("c1_random_n10k", "bcrp", n, src, dst, act, 4)


def c2_kripke(n: int = 1_000_000, out_degree: int = 5, colours: int = 4, seed: int = 2) -> Instance:
    """c2: RCPP Kripke structure, fixed out-degree, uniform targets, pi0 a
    uniform 4-colouring (2 atomic propositions) in canonical leader form."""
    g = np.random.default_rng(seed)
    src = np.repeat(np.arange(n, dtype=np.int32), out_degree)
    dst = g.integers(0, n, size=n * out_degree, dtype=np.int32)
    colour = g.integers(0, colours, size=n)
    return Instance(f"c2_kripke_n{n}", "rcpp", n, _i32(src), _i32(dst), pi0=canonical(colour))


def chain(n: int = 200_000) -> Instance:
    """c3: chain 0 -> 1 -> ... -> n-1, one label: BCRP needs 2n-2 rounds."""
    src = np.arange(n - 1, dtype=np.int32)
    return Instance(f"c3_chain_n{n}", "bcrp", n, src, src + 1, np.zeros(n - 1, np.int32), 1,
                    truth=np.arange(n, dtype=np.int32), expect_supersteps=2 * n - 2)


def fanout(n: int) -> Instance:
    """Fan_out family (cli.py:62-75): a chain over 2..n-1 labelled a, and two
    hubs with b-edges to every state."""
    if n < 3:
        raise ValueError("fan-out family needs n >= 3")
    chain_src = np.arange(2, n - 1, dtype=np.int32)
    hubs = np.repeat(np.array([0, 1], np.int32), n)
    targets = np.tile(np.arange(n, dtype=np.int32), 2)
    src = np.concatenate([chain_src, hubs])
    dst = np.concatenate([chain_src + 1, targets])
    act = np.concatenate([np.zeros(chain_src.size, np.int32), np.ones(2 * n, np.int32)])
    return Instance(f"fanout_{n}", "bcrp", n, _i32(src), _i32(dst), _i32(act), 2)


def c4_uniform(n: int = 5_000_000, m: int = 50_000_000, num_actions: int = 256,
               seed: int = 4) -> Instance:
    """c4(i): iid uniform (source, label, target) with 256 labels."""
    g = np.random.default_rng(seed)
    src = g.integers(0, n, size=m, dtype=np.int32)
    act = g.integers(0, num_actions, size=m, dtype=np.int32)
    dst = g.integers(0, n, size=m, dtype=np.int32)
    return Instance(f"c4_uniform_n{n}", "bcrp", n, src, dst, act, num_actions)


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (element-wise, uint64)."""
    z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def signature_bisim(n: int, src, act, dst, max_iter: int = 100_000, init=None) -> np.ndarray:
    """Coarsest bisimulation by iterated signature refinement: the class of s
    is refined by the set {(a, class(t)) : s -a-> t} until the number of
    classes stops growing (starting from ``init`` classes if given, else
    the trivial partition).  Independent of the PRAM algorithm; set hashing is
    64-bit (collisions would only merge, and are checked by the caller's
    stability test)."""
    src = np.asarray(src, np.int64)
    act = np.asarray(act, np.int64)
    dst = np.asarray(dst, np.int64)
    cls = np.zeros(n, np.int64) if init is None else np.unique(np.asarray(init), return_inverse=True)[1].reshape(-1).astype(np.int64)
    count = int(cls.max()) + 1
    k2 = np.uint64(0xC2B2AE3D27D4EB4F)
    A = int(act.max()) + 1 if act.size else 1
    K = np.int64(A * (n + 1))               # pair = act*(n+1) + class < K
    if (n + 1) * int(K) >= 2 ** 62:
        raise ValueError("instance too large for signature_bisim's packed keys")
    for _ in range(max_iter):
        pair = act * (n + 1) + cls[dst]
        key = np.unique(src * K + pair) if src.size else np.zeros(0, np.int64)
        s_of = key // K
        p_of = (key % K).astype(np.uint64)
        h = _mix64(p_of)
        sig = np.zeros(n, np.uint64)
        np.add.at(sig, s_of, h)
        sig2 = np.zeros(n, np.uint64)
        np.bitwise_xor.at(sig2, s_of, _mix64(h ^ k2))
        combo = np.stack([cls.astype(np.uint64), sig, sig2], axis=1)
        _, inv = np.unique(combo, axis=0, return_inverse=True)
        inv = inv.reshape(-1).astype(np.int64)
        new_count = int(inv.max()) + 1
        cls = inv
        if new_count == count:
            break
        count = new_count
    return canonical(cls)


def lifted_quotient(n: int, k: int, num_actions: int, templates: int, labels_per_template: int,
                    edges_per_label: int, seed: int, name: str = "lifted") -> Instance:
    """Lifted-quotient LTS with exact ground truth.

    A small quotient Q (k states) draws each state's label set from a pool of
    templates and ``edges_per_label`` random targets per label.  Each
    Q-state is lifted to c = n // k copies; every copy repeats its Q-state's
    edges, each redirected to a random copy of the Q-target, and state ids
    are randomly permuted.  The projection copy -> Q-state is a functional
    bisimulation, so the coarsest bisimulation of the lift is the pull-back
    of Q's: ground truth costs one refinement of Q.
    """
    if n % k:
        raise ValueError("n must be a multiple of k")
    c = n // k
    g = np.random.default_rng(seed)
    pool = np.stack([np.sort(g.choice(num_actions, size=labels_per_template, replace=False))
                     for _ in range(templates)])
    tmpl = g.integers(0, templates, size=k)
    deg = labels_per_template * edges_per_label
    q_src = np.repeat(np.arange(k, dtype=np.int64), deg)
    q_act = np.repeat(pool[tmpl], edges_per_label, axis=1).reshape(-1).astype(np.int64)
    q_dst = g.integers(0, k, size=k * deg, dtype=np.int64)
    q_truth = signature_bisim(k, q_src, q_act, q_dst)
    perm = g.permutation(n).astype(np.int64)          # lifted (q, i) -> state id perm[q*c+i]
    mq = q_src.size
    copies = np.arange(c, dtype=np.int64)
    # transition (e, i): Q-edge e lifted at copy i, target copy drawn uniformly
    src = perm[(q_src[:, None] * c + copies[None, :]).reshape(-1)].astype(np.int32)
    tcopy = g.integers(0, c, size=mq * c, dtype=np.int64)
    dst = perm[(np.repeat(q_dst, c) * c + tcopy)].astype(np.int32)
    act = np.repeat(q_act, c).astype(np.int32)
    # ground truth: class of state id = Q-class of its Q-state
    q_of_id = np.empty(n, np.int64)
    q_of_id[perm] = np.arange(n, dtype=np.int64) // c
    truth = canonical(q_truth[q_of_id])
    return Instance(name, "bcrp", n, src, dst, act, num_actions, truth=truth)


def c4_lifted(n: int = 5_000_000, k: int = 20_000, seed: int = 44) -> Instance:
    """c4(ii): |Act| = 256, m = 10 n, label sets from 6 templates x 5 labels."""
    return lifted_quotient(n, k, 256, templates=6, labels_per_template=5, edges_per_label=2,
                           seed=seed, name=f"c4_lifted_n{n}")


def c5_vlts(n: int = 10_000_000, k: int = 5_000, seed: int = 0) -> Instance:
    """c5: VLTS-shaped lifted quotient, n = 10M, m = 100M (out-degree 10),
    |Act| = 32, <= k blocks (blocks/n ~ 5e-4)."""
    return lifted_quotient(n, k, 32, templates=8, labels_per_template=5, edges_per_label=2,
                           seed=seed, name=f"c5_vlts_n{n}_seed{seed}")


def is_stable(n: int, src, act, dst, block) -> bool:
    """Every block is stable under every block (oracle.py:128-141 restated
    with arrays): every state sees the same set of (action, target block)
    pairs as its leader.  Sets are compared by size and a 64-bit sum-hash."""
    block = np.asarray(block, np.int64)
    src = np.asarray(src, np.int64)
    act = np.asarray(act, np.int64)
    A = int(act.max()) + 1 if act.size else 1
    K = np.int64(A * (n + 1))
    if (n + 1) * int(K) >= 2 ** 62:
        raise ValueError("instance too large for is_stable's packed keys")
    key = np.unique(src * K + act * (n + 1) + block[np.asarray(dst, np.int64)])
    s = key // K
    p = (key % K).astype(np.uint64)
    cnt = np.bincount(s, minlength=n)
    if np.any(cnt != cnt[block]):
        return False
    h = _mix64(p)
    f = np.zeros(n, np.uint64)
    np.add.at(f, s, h)
    return bool(np.all(f == f[block]))
