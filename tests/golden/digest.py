"""Digest helper shared by the golden generator and the tests."""

import hashlib

import numpy as np


def digest(a):
    if a is None:
        return None
    a = np.asarray(a, dtype="<f8")
    return hashlib.sha256(a.tobytes(order="F")).hexdigest()


def unhex(s):
    return float.fromhex(s)
