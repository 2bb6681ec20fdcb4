"""Synthetic planted-block power-law graphs.

Input generation shared by both bench arms, so the GPU engine and the
reference CPU engine train on byte-identical graphs.  It loads only
``synth/_build/libqgnn_synth.so`` (built by ``synth/Makefile``): neither the
product library nor the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "_build", "libqgnn_synth.so")


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    if not os.path.exists(SO):
        build()
    L = C.CDLL(SO)
    i64, dbl, vp = C.c_int64, C.c_double, C.c_void_p
    L.qgnn_synth_planted.restype = C.c_int
    L.qgnn_synth_planted.argtypes = [i64, i64, i64, i64, i64, dbl, dbl, dbl, C.c_uint64] + [vp] * 7
    return L


_L = None


def generate_planted(nodes: int, n_edges: int, feat: int, classes: int, blocks: int,
                     cross_frac: float, gamma: float = 2.5, sep: float = 1.0, seed: int = 1):
    """Planted-block power-law graph: symmetric sorted CSR (``adj_ptr`` int64,
    ``adj`` int32, exactly 2*n_edges entries), fp32 ``features``
    (sep*mu_class + N(0,1)), ``labels``, 60/20/20 ``train``/``val``/``test``
    masks, and ``owner`` = the planted block of every node (contiguous id
    ranges)."""
    global _L
    if _L is None:
        _L = _load()
    g = dict(adj_ptr=np.zeros(nodes + 1, np.int64), adj=np.zeros(2 * n_edges, np.int32),
             features=np.zeros((nodes, feat), np.float32), labels=np.zeros(nodes, np.int32),
             train=np.zeros(nodes, np.uint8), val=np.zeros(nodes, np.uint8),
             test=np.zeros(nodes, np.uint8))
    st = _L.qgnn_synth_planted(nodes, n_edges, feat, classes, blocks, cross_frac, gamma, sep,
                               seed, *(g[k].ctypes.data for k in ("adj_ptr", "adj", "features",
                                                                  "labels", "train", "val",
                                                                  "test")))
    if st != 0:
        raise ValueError(f"generate_planted: bad arguments (status {st})")
    g["owner"] = (np.arange(nodes, dtype=np.int64) // (-(-nodes // blocks))).astype(np.uint32)
    return g
