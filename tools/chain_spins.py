"""Carry-poll statistics of the chain kernel's pass 1 (ODX_CHAIN_KNOB=4 + ODX_CHAIN_TRACE):
    ODX_CHAIN_KNOB=4 ODX_CHAIN_TRACE=/tmp/tr.bin python tools/cfg5_time.py --reps 1 --check-n 0
    python tools/chain_spins.py /tmp/tr.bin
Counts are per warp (lane 0 of every compute warp adds its own)."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64, count=3)
print(f"warp-level applies {a[2]}, late carries {a[1]} ({100.0 * a[1] / max(a[2], 1):.1f}%), "
      f"reloads {a[0]} ({a[0] / max(a[2], 1):.2f} per apply)")
