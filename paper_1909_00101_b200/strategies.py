"""Parallel pivot orderings and the multi-GPU block schedule.

``gen_table`` / ``validate_table`` / ``comm_mapping`` reproduce the
reference's tables exactly (strategies.py:45-143): ME is the round-robin
(circle-method) tournament with every step's pairs sorted, MM the modified
modulus ordering.  The device library builds the same tables natively
(csrc/hzg_api.cu); ``tests/test_strategies.py`` checks both against the
oracle.

For several GPUs the *pair sets* of each ME step stay exactly the
reference's, but pairs are assigned to GPUs by their circle-method position
(``circle_positions``): position i of step k holds the pair
(line[i], line[N-1-i]) with line = [0, rotate(others, k)].  Between steps
every block moves by at most one position, so with contiguous position
ranges per GPU only O(1) blocks cross a GPU boundary per step
(``block_schedule``).
"""

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np


@dataclass
class StrategyTable:
    order: int
    kind: str
    steps: List[List[Tuple[int, int]]]

    def as_array(self):
        """Steps as an int32 array of shape (steps, order//2, 2)."""
        return np.asarray(self.steps, dtype=np.int32)


@dataclass
class CommMapping:
    """entries[k][r] = (p, q, t0, t1) for step k and holder r."""

    order: int
    steps: int
    entries: List[List[Tuple[int, int, int, int]]]


def _circle_lines(n):
    """The circle-method line of every ME step: line[0] = 0 is fixed, the
    other n-1 indices rotate right by one per step."""
    ring = list(range(1, n))
    for _ in range(n - 1):
        yield [0] + ring
        ring = ring[-1:] + ring[:-1]


def circle_positions(n):
    """(steps, n/2, 2) int array: pair at circle position i of each ME step,
    ordered (min, max).  As sets, row k equals gen_table('me', n).steps[k]."""
    half = n // 2
    out = np.empty((n - 1, half, 2), dtype=np.int64)
    for k, line in enumerate(_circle_lines(n)):
        for i in range(half):
            a, b = line[i], line[n - 1 - i]
            out[k, i] = (min(a, b), max(a, b))
    return out


def gen_table(kind, n):
    """Strategy table of the given kind for even n >= 2 (strategies.py:45-56)."""
    if n < 2 or n % 2 != 0:
        raise ValueError("strategy order must be even and at least 2, got %r" % (n,))
    kind = kind.lower()
    if kind == "me":
        steps = [sorted(map(tuple, row.tolist())) for row in circle_positions(n)]
    elif kind == "mm":
        steps = _modified_modulus(n)
    else:
        raise ValueError("unknown strategy kind %r" % (kind,))
    return StrategyTable(n, kind, steps)


def _modified_modulus(n):
    """Step k pairs i with (k - i) mod n; for even k the two fixed points
    k/2 and k/2 + n/2 of that involution are paired together."""
    half = n // 2
    steps = []
    for k in range(n):
        used = [False] * n
        pairs = []
        for i in range(n):
            j = (k - i) % n
            if used[i] or j == i or used[j]:
                continue
            used[i] = used[j] = True
            pairs.append((min(i, j), max(i, j)))
        if k % 2 == 0 and not used[k // 2]:
            a, b = k // 2, k // 2 + half
            pairs.append((min(a, b), max(a, b)))
        steps.append(sorted(pairs))
    return steps


def validate_table(t):
    """Exhaustive disjointness / coverage / cyclicity check (strategies.py:96-114)."""
    n = t.order
    want = {(i, j) for i in range(n) for j in range(i + 1, n)}
    seen = []
    disjoint_ok = True
    for step in t.steps:
        used = set()
        for (i, j) in step:
            if i in used or j in used or not (0 <= i < j < n):
                disjoint_ok = False
            used.update((i, j))
        disjoint_ok &= len(step) == n // 2
        seen.extend(step)
    coverage_ok = set(seen) == want
    return {"cyclic": coverage_ok and len(seen) == len(want), "coverage_ok": coverage_ok,
            "disjoint_ok": disjoint_ok}


def _dest(step, stripe):
    for rank, (i, j) in enumerate(step):
        if i == stripe:
            return -(rank + 1)
        if j == stripe:
            return rank + 1
    raise ValueError("stripe %d absent from step %r" % (stripe, step))


def comm_mapping(t):
    """Route each holder's two stripes to the holder that needs them in the
    next step; rank d at its first slot encodes -(d+1), second slot +(d+1)
    (strategies.py:117-143)."""
    s = len(t.steps)
    entries = []
    for k in range(s):
        nxt = t.steps[(k + 1) % s]
        entries.append([(p, q, _dest(nxt, p), _dest(nxt, q)) for (p, q) in t.steps[k]])
    return CommMapping(t.order, s, entries)


def dump_table(t, mapping=None):
    """Text form: one step per line, pairs as i-j (strategies.py:146-155)."""
    lines = []
    for k, step in enumerate(t.steps):
        lines.append(" ".join("%d-%d" % (i, j) for (i, j) in step))
        if mapping is not None:
            lines.append("  " + " ".join("r%d:p%d,q%d,t0=%+d,t1=%+d" % (r, p, q, t0, t1)
                                         for r, (p, q, t0, t1) in enumerate(mapping.entries[k])))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# multi-GPU block schedule
# ---------------------------------------------------------------------------

def slot_ranges(npos, nranks):
    """Contiguous circle-position ranges [lo, hi) per rank, sizes differing by <= 1."""
    base, extra = divmod(npos, nranks)
    out, lo = [], 0
    for r in range(nranks):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def weighted_slot_ranges(npos, nranks, end_weight=1.0):
    """Contiguous circle-position ranges [lo, hi) per rank with the two end
    ranks weighted by ``end_weight`` relative to the interior ranks (every
    rank keeps at least one position).  The positions next to the ends of
    the circle ordering need more inner sweeps per pair, so
    giving their ranks fewer pairs balances the per-step time; the pairs
    and per-pair work are unchanged, so results do not depend on it."""
    if nranks < 3 or end_weight == 1.0:
        return slot_ranges(npos, nranks)
    wts = [end_weight] + [1.0] * (nranks - 2) + [end_weight]
    tot = sum(wts)
    cuts = [0]
    acc = 0.0
    for r in range(nranks - 1):
        acc += wts[r]
        cuts.append(int(round(npos * acc / tot)))
    cuts.append(npos)
    for r in range(1, nranks):                # at least one position per rank
        cuts[r] = max(cuts[r], cuts[r - 1] + 1)
    for r in range(nranks - 1, 0, -1):
        cuts[r] = min(cuts[r], cuts[r + 1] - 1)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def owner_of_blocks(nblk, nranks):
    """owner[k][b]: rank holding block b during ME step k (circle positions,
    contiguous position ranges per rank)."""
    pos = circle_positions(nblk)
    ranges = slot_ranges(nblk // 2, nranks)
    owner = np.empty((nblk - 1, nblk), dtype=np.int64)
    for r, (lo, hi) in enumerate(ranges):
        for i in range(lo, hi):
            owner[:, pos[:, i, 0]] = -1  # placeholder, overwritten below
    for k in range(nblk - 1):
        for r, (lo, hi) in enumerate(ranges):
            for i in range(lo, hi):
                owner[k, pos[k, i, 0]] = r
                owner[k, pos[k, i, 1]] = r
    return owner


def block_moves(nblk, nranks):
    """For every step transition k -> k+1 (cyclic), the list of
    (block, src_rank, dst_rank) whose owner changes."""
    own = owner_of_blocks(nblk, nranks)
    steps = nblk - 1
    moves = []
    for k in range(steps):
        a, b = own[k], own[(k + 1) % steps]
        moves.append([(int(blk), int(a[blk]), int(b[blk])) for blk in np.nonzero(a != b)[0]])
    return moves
