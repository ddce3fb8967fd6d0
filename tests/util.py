"""Shared helpers for the test-suite (golden fixtures, limb conversions)."""
import json
import os

import numpy as np

from oracle.refshim import cols_to_ints, ints_to_cols  # noqa: F401

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CURVE_IDS = {"sm2": 0, "secp256k1": 1}


def golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def hex_cols(hs):
    return ints_to_cols([int(h, 16) for h in hs])


def cols_hex(cols):
    return [format(v, "064x") for v in cols_to_ints(cols)]


def pts_from_hex(d):
    return hex_cols(d["x"]), hex_cols(d["y"]), np.array(d["inf"], np.uint8)


def pts_to_hex(P):
    return dict(x=cols_hex(P[0]), y=cols_hex(P[1]), inf=[int(v) for v in P[2]])


def wide_cols(hs):
    """128-hex-digit strings -> (16, n) uint32 columns"""
    out = np.zeros((16, len(hs)), np.uint32)
    for i, h in enumerate(hs):
        t = int(h, 16)
        for k in range(16):
            out[k, i] = (t >> (32 * k)) & 0xFFFFFFFF
    return out
