"""Seeded degree-corrected SBM arc lists and stream slicings (input generators).

These produce the synthetic stand-ins for the Graph Challenge datasets that
BASELINE.json's configs name (SURVEY.md §8(d) "Inputs"). The reference has no
DC-SBM (its ``sbm.py`` is a Bernoulli planted partition), so
nothing here needs parity: the same arc array is fed to the reference/oracle
and to the device path. Generation is host numpy and never on the timed path.

Model
-----
* block proportions ``pi ~ Dirichlet(alpha * 1_B)``; vertex labels ``z_i ~ pi``;
* vertex propensity ``theta_i`` from a power law with exponent ``-gamma``
  truncated to ``[dmin, dmax]`` (inverse-CDF sampling);
* ``M`` directed arcs: the source is drawn proportional to ``theta``; with
  probability ``r / (r + 1)`` the destination is drawn proportional to
  ``theta`` inside the source's block, otherwise proportional to ``theta``
  among the vertices of all *other* blocks;
* duplicates and self-loops are kept, so ``from_edges`` has real work to do.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["DcsbmSpec", "CONFIGS", "generate_dcsbm", "emerging_slices", "snowball_slices"]


@dataclass(frozen=True)
class DcsbmSpec:
    n: int
    blocks: int
    arcs: int
    alpha: float = 3.0
    ratio: float = 5.0
    gamma: float = 2.5
    dmin: float = 10.0
    dmax: float = 100.0
    seed: int = 0


# BASELINE.json configs[0..3]; C5 streams C2.
CONFIGS = {
    "c1": DcsbmSpec(n=5_000, blocks=19, arcs=100_000, alpha=3.0, ratio=5.0),
    "c2": DcsbmSpec(n=50_000, blocks=44, arcs=1_000_000, alpha=1.0, ratio=2.0),
    "c3": DcsbmSpec(n=500_000, blocks=98, arcs=10_000_000, alpha=3.0, ratio=5.0),
    "c4": DcsbmSpec(n=2_000_000, blocks=160, arcs=40_000_000, alpha=3.0, ratio=5.0),
}


def _power_law(rng, size, gamma, lo, hi):
    """Inverse-CDF draw from p(x) ~ x^-gamma on [lo, hi]."""
    e = 1.0 - gamma
    u = rng.random(size)
    return (lo**e + u * (hi**e - lo**e)) ** (1.0 / e)


def generate_dcsbm(spec: DcsbmSpec):
    """Return ``(edges (M,2) int64, truth labels (n,) int64)``."""
    rng = np.random.default_rng(spec.seed)
    n, nb = spec.n, spec.blocks
    pi = rng.dirichlet(np.full(nb, spec.alpha))
    z = rng.choice(nb, size=n, p=pi)
    theta = _power_law(rng, n, spec.gamma, spec.dmin, spec.dmax)

    # vertices grouped by block; cumulative propensity in that order
    order = np.argsort(z, kind="stable")
    theta_sorted = theta[order]
    cum = np.cumsum(theta_sorted)
    counts = np.bincount(z, minlength=nb)
    starts = np.concatenate([[0], np.cumsum(counts)])
    cum0 = np.concatenate([[0.0], cum])  # cum0[i] = sum of first i sorted thetas
    block_lo = cum0[starts[:-1]]
    block_mass = cum0[starts[1:]] - block_lo
    total = cum0[-1]

    m = spec.arcs
    src = np.searchsorted(cum, rng.random(m) * total, side="right")
    src = np.minimum(src, n - 1)
    src_v = order[src]
    zb = z[src_v]
    inside = rng.random(m) < spec.ratio / (spec.ratio + 1.0)

    # destination block: own block, or another block proportional to its mass
    u = rng.random(m)
    other_mass = total - block_mass[zb]
    pos = u * other_mass
    # skip the source's own block in the cumulative block-mass scale
    pos = np.where(pos >= block_lo[zb], pos + block_mass[zb], pos)
    blk_cum = np.cumsum(block_mass)
    other_b = np.minimum(np.searchsorted(blk_cum, pos, side="right"), nb - 1)
    dst_b = np.where(inside, zb, other_b)

    v = rng.random(m)
    target = block_lo[dst_b] + v * block_mass[dst_b]
    dst = np.searchsorted(cum, target, side="right")
    dst = np.clip(dst, starts[dst_b], np.maximum(starts[dst_b + 1] - 1, starts[dst_b]))
    dst_v = order[dst]
    edges = np.column_stack([src_v, dst_v]).astype(np.int64)
    return edges, z.astype(np.int64)


def emerging_slices(edges: np.ndarray, stages: int, seed: int):
    """Config 5(a): a seeded random permutation of the arcs cut into equal slices."""
    perm = np.random.default_rng((seed, 1)).permutation(len(edges))
    return [edges[c] for c in np.array_split(perm, stages)]


def snowball_slices(edges: np.ndarray, n: int, stages: int, seed: int, roots: int = 10):
    """Config 5(b): BFS admission from seeded roots, vertices renumbered by admission.

    Returns ``(relabel, [(delta_edges, n_after), ...])``: old vertices form a
    prefix of the new numbering (as partition_stream requires) and each stage
    receives the arcs whose later-admitted endpoint joins at that stage.
    """
    rng = np.random.default_rng((seed, 2))
    src, dst = edges[:, 0], edges[:, 1]
    both = np.concatenate([src, dst])
    other = np.concatenate([dst, src])
    idx = np.argsort(both, kind="stable")
    nbr = other[idx]
    offs = np.concatenate([[0], np.cumsum(np.bincount(both, minlength=n))])
    admit = np.full(n, -1, dtype=np.int64)
    queue = list(rng.choice(n, size=min(roots, n), replace=False))
    for r in queue:
        admit[r] = 0
    order = []
    head = 0
    while head < len(queue) or len(order) < n:
        if head == len(queue):  # disconnected remainder: restart from a fresh vertex
            rest = np.flatnonzero(admit < 0)
            queue.append(int(rest[0]))
            admit[rest[0]] = 0
        v = int(queue[head])
        head += 1
        order.append(v)
        for w in nbr[offs[v] : offs[v + 1]]:
            if admit[w] < 0:
                admit[w] = 0
                queue.append(int(w))
    order = np.asarray(order, dtype=np.int64)
    relabel = np.empty(n, dtype=np.int64)
    relabel[order] = np.arange(n)
    bounds = np.linspace(0, n, stages + 1).round().astype(np.int64)
    e = relabel[edges]
    later = e.max(axis=1)
    stage_of = np.searchsorted(bounds[1:], later, side="right")
    out = []
    for s in range(stages):
        out.append((e[stage_of == s], int(bounds[s + 1])))
    return relabel, out
