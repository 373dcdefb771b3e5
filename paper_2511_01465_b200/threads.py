"""Host-thread control, mirroring odescan.threads (threads.py:17-32).

The reference clamps numba's worker count for its CPU kernels.  Here the
compute runs on the GPU; the only host-side parallel work on the solve path is
odx_solve_host's staging copy of pageable numpy buffers, so these functions
size that pool: max_threads() is the pool size fixed at first use
(ODX_HOST_THREADS, default min(8, cores/2)), set_threads(n) clamps n into
[1, max_threads()], applies it and returns the value used — the reference's
contract.
"""

from __future__ import annotations

import os

__all__ = ["max_threads", "set_threads", "hardware_threads"]


def max_threads() -> int:
    """Upper bound on usable host copy threads for this process."""
    from . import _native
    return int(_native.lib().odx_host_threads_max())


def hardware_threads() -> int:
    """Hardware threads the host reports."""
    return os.cpu_count() or 1


def set_threads(n: int) -> int:
    """Clamp n into [1, max_threads()], apply it, and return the value used."""
    from . import _native
    return int(_native.lib().odx_set_host_threads(int(n)))
