"""Affine-map element algebra (the scan operator) and list-based scans.

Mirrors odescan.affine_scan (/root/reference/pkg/src/odescan/affine_scan.py):
AffineElement (:35-57), identity (:60-62), combine(earlier, later) =
(F_l F_e, F_l c_e + c_l) (:64-78), init_elements (:81-105), scan_sequential
(:108-115), scan_parallel (:117-155), extract_states (:158-164) and the array
converters.  These list-based forms are small host utilities kept for API
compatibility; the array scan the solver runs is the device kernel
(kernels.scan_affine / the fused solve).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["AffineElement", "identity", "combine", "init_elements", "scan_sequential",
           "scan_parallel", "extract_states", "elements_to_arrays", "arrays_to_elements"]


@dataclass(frozen=True, eq=False)
class AffineElement:
    """The map z -> F z + c."""

    F: np.ndarray
    c: np.ndarray

    def __post_init__(self):
        F = np.asarray(self.F, dtype=np.float64)
        c = np.asarray(self.c, dtype=np.float64)
        if F.ndim != 2 or F.shape[0] != F.shape[1]:
            raise ValueError(f"F must be square, got shape {F.shape}")
        if c.shape != (F.shape[0],):
            raise ValueError(f"c must be a vector matching F: F is {F.shape}, c is {c.shape}")
        object.__setattr__(self, "F", F)
        object.__setattr__(self, "c", c)

    @property
    def dim(self) -> int:
        return self.F.shape[0]


def identity(dim: int) -> AffineElement:
    return AffineElement(np.eye(dim), np.zeros(dim))


def combine(earlier: AffineElement, later: AffineElement) -> AffineElement:
    """Apply `earlier` first, then `later`."""
    if earlier.dim != later.dim:
        raise ValueError(f"dimension mismatch: earlier is {earlier.dim}-dim, "
                         f"later is {later.dim}-dim")
    return AffineElement(later.F @ earlier.F, later.F @ earlier.c + later.c)


def init_elements(F_seq, c_seq, z0) -> list:
    """Elements whose inclusive scan gives z_1..z_N; element 0 absorbs z0 (F := 0)."""
    if len(F_seq) != len(c_seq):
        raise ValueError(f"F_seq and c_seq lengths differ: {len(F_seq)} vs {len(c_seq)}")
    if len(F_seq) == 0:
        raise ValueError("need at least one step")
    z0 = np.asarray(z0, dtype=np.float64)
    F0 = np.asarray(F_seq[0], dtype=np.float64)
    if z0.shape != (F0.shape[0],):
        raise ValueError(f"z0 has shape {z0.shape}, expected ({F0.shape[0]},)")
    first = AffineElement(np.zeros_like(F0), F0 @ z0 + np.asarray(c_seq[0], np.float64))
    return [first] + [AffineElement(F, c) for F, c in zip(F_seq[1:], c_seq[1:])]


def scan_sequential(elements) -> list:
    if len(elements) == 0:
        raise ValueError("cannot scan an empty sequence")
    out = [elements[0]]
    for e in elements[1:]:
        out.append(combine(out[-1], e))
    return out


def scan_parallel(elements, combine_fn=combine) -> list:
    """Inclusive scan with logarithmic combine depth (Hillis-Steele doubling)."""
    n = len(elements)
    if n == 0:
        raise ValueError("cannot scan an empty sequence")
    cur = list(elements)
    shift = 1
    while shift < n:
        cur = [cur[k] if k < shift else combine_fn(cur[k - shift], cur[k]) for k in range(n)]
        shift *= 2
    return cur


def extract_states(prefixes) -> list:
    return [p.c for p in prefixes]


def elements_to_arrays(elements):
    F = np.stack([e.F for e in elements])
    c = np.stack([e.c for e in elements])
    return F, c


def arrays_to_elements(F, c):
    return [AffineElement(F[k].copy(), c[k].copy()) for k in range(c.shape[0])]
