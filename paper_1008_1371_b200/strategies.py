"""Modified-modulus pivot stepper (/root/reference/pkg/src/hjsvd/
strategies.py:20-72).  The solver keeps the stepper quadruples on the device
and advances them inside the step kernel; these host objects mirror the
reference's API (stepper_advance_all runs the device kernel)."""

from dataclasses import dataclass

import numpy as np

from . import _device
from .errors import ShapeError


@dataclass
class StepperState:
    """Per-block stepper quadruples (strategies.py:20-38)."""

    r: int
    ip: np.ndarray
    jp: np.ndarray
    iblk: np.ndarray
    jblk: np.ndarray

    def pairs(self):
        lo = np.minimum(self.iblk, self.jblk)
        hi = np.maximum(self.iblk, self.jblk)
        return [(int(i), int(j)) for i, j in zip(lo, hi)]


def stepper_init(r):
    """Antidiagonal start: block k holds the pair (k, r-k-1) (strategies.py:41-47)."""
    if r < 2 or r % 2 != 0:
        raise ShapeError("r must be even and >= 2")
    b = r // 2
    k = np.arange(b, dtype=np.int64)
    return StepperState(r, k.copy(), r - k - 1, k.copy(), r - k - 1)


def stepper_advance(state, k):
    """Advance block k (strategies.py:50-66): ip + jp >= r - 1 branch."""
    r = state.r
    if state.ip[k] + state.jp[k] >= r - 1:
        state.ip[k] += 1
        if state.ip[k] == state.jp[k]:
            state.ip[k] -= r // 2
            state.jp[k] = state.ip[k]
        state.iblk[k] = state.ip[k]
    else:
        state.jp[k] += 1
        state.jblk[k] = state.jp[k]
    return state


def stepper_advance_all(state):
    """Advance every block by one step on the device (strategies.py:69-72)."""
    _device.advance_stepper(state.ip, state.jp, state.iblk, state.jblk, state.r)
    return state


def schedule_table(r, steps):
    """Host enumeration of `steps` consecutive steps' slot pairs (i, j), as an
    int64 array (steps, r/2, 2) -- used by the block driver's multi-GPU
    planner and the tests; pure integer bookkeeping."""
    S = stepper_init(r)
    out = np.empty((steps, r // 2, 2), dtype=np.int64)
    for s in range(steps):
        out[s, :, 0] = np.minimum(S.iblk, S.jblk)
        out[s, :, 1] = np.maximum(S.iblk, S.jblk)
        for k in range(r // 2):
            stepper_advance(S, k)
    return out
