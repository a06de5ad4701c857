"""Solver configuration (the reference's SolverConfig, pointwise.py:40-81).

Same fields, defaults, decoding and ValueError behaviour.  Three B200-only
fields are added:

* ``exact`` selects the reference-order Grammian and postmultiply kernels
  (bitwise agreement with the CPU reference) instead of the FP64
  tensor-core (DMMA) kernels used by default;
* ``approx_2x2`` (DMMA mode, default on) computes the 2x2 transforms with
  the short-chain forms (reciprocal square roots of sums of squares instead
  of the reference's chain of divisions and square roots; tolerance
  parity, hzg_device.cuh).  Off, or with ``exact``, the 2x2 math is
  bitwise the reference's;
* ``split_rows`` (DMMA mode) fixes the rows per Grammian split (a multiple
  of 64, 0 = the default geometry).  The split geometry sets the summation
  order of the block Grammians, so it is part of the configuration, not of
  the environment: results are bitwise reproducible for a given
  SolverConfig, whatever HZG_* performance variables are set.
"""

from dataclasses import dataclass, field as dc_field

EPS = 2.0 ** -52


@dataclass
class SolverConfig:
    """Solver variant selection.

    variant_id decodes as: convergence criterion C1 for ids < 4 and C2
    otherwise; ids 0, 1, 4, 5 prescale the columns once (unit G column norms)
    while 2, 3, 6, 7 rescale each pivot pair on the fly; odd ids use the
    compensated dot products.
    """

    variant_id: int = 0
    outer_kind: str = "me"
    inner_kind: str = "me"
    blocking: str = "fb"
    sorting: bool = True
    max_inner_sweeps: int = 0
    max_outer_sweeps: int = 30
    block_width: int = 8
    gate_eps: float = EPS
    fallback_qr: bool = True
    shorten: str = "grammian"
    pool: int = 1
    exact: bool = False
    split_rows: int = 0
    approx_2x2: bool = True
    criterion: str = dc_field(init=False, default="C1")
    prescale: bool = dc_field(init=False, default=True)
    compensated: bool = dc_field(init=False, default=False)

    def __post_init__(self):
        if self.variant_id not in range(8):
            raise ValueError("variant_id must be 0..7")
        if self.blocking not in ("fb", "bo"):
            raise ValueError("blocking must be fb or bo")
        if self.outer_kind not in ("me", "mm") or self.inner_kind not in ("me", "mm"):
            raise ValueError("strategy kinds must be me or mm")
        if self.shorten not in ("grammian", "qr"):
            raise ValueError("shorten must be grammian or qr")
        if self.block_width < 1:
            raise ValueError("block width must be at least 1")
        if self.split_rows < 0 or self.split_rows % 64:
            raise ValueError("split_rows must be 0 or a positive multiple of 64")
        self.criterion = "C1" if self.variant_id < 4 else "C2"
        self.prescale = self.variant_id in (0, 1, 4, 5)
        self.compensated = self.variant_id % 2 == 1
        if self.max_inner_sweeps <= 0:
            self.max_inner_sweeps = 30 if self.blocking == "fb" else 1


@dataclass
class SweepStats:
    """Applied-transformation counters (pointwise.py:84-93)."""

    total: int = 0
    big: int = 0

    def __post_init__(self):
        if self.big > self.total:
            raise ValueError("big count cannot exceed the total")
