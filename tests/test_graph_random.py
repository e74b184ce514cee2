"""Randomized bit-exactness of the library's graph ordering against the oracle.

The product's Tarjan / exact FAS / weighted Eades-Lin-Smyth / min-heap Kahn
(hsw_host.cpp, written independently of oracle/hosweep_oracle.cpp) is compared
with the oracle on random weighted digraphs, in the spirit of the reference's
own randomized graph tests (test_sweepgraph.cpp:119-151: Tarjan vs reachability
on 1000 graphs, exact DP vs n! brute force on 500 graphs): orders, cut sets and
cut weights must be identical, including ties (integer weights from small sets),
SCCs on both sides of the exact-FAS threshold, self-consistent multi-edges.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1810_11080_b200 import _capi


def _product_order(nv, edges, w, thr):
    L = _capi.load()
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    w = np.ascontiguousarray(np.asarray(w, np.float64))
    order = np.zeros(nv, np.int32)
    lag = np.zeros(max(len(w), 1), np.int32)
    lw = C.c_double()
    n = L.hsw_debug_graph_order(nv, e.shape[0], e.ctypes.data if len(w) else None,
                                w.ctypes.data if len(w) else None, thr, order.ctypes.data, lag.ctypes.data,
                                C.byref(lw))
    assert n >= 0, _capi.last_error()
    return list(order), list(lag[:n]), lw.value


def _random_graph(rng):
    nv = int(rng.integers(1, 48))
    kind = rng.integers(0, 3)
    p = [0.04, 0.12, 0.35][kind]
    edges = []
    for a in range(nv):
        for b in range(nv):
            if a != b and rng.random() < p:
                edges.append((a, b))
    rng.shuffle(edges)
    if rng.random() < 0.5:   # ties: a few distinct weights
        w = rng.choice(np.array([0.5, 1.0, 1.0, 2.0, 3.0]), size=len(edges))
    else:
        w = rng.uniform(0.01, 5.0, size=len(edges))
    return nv, edges, w


@pytest.mark.parametrize("seed", range(6))
def test_random_graphs_order_cut_set_and_weight_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(100):
        nv, edges, w = _random_graph(rng)
        thr = int(rng.choice([3, 10, 22] if nv <= 18 else [3, 10]))   # 2^22-state DPs only on small graphs
        got = _product_order(nv, edges, w, thr)
        ref = O.graph_order(nv, edges, w, 2, thr)
        assert list(got[0]) == list(ref[0]), (nv, len(edges), thr)
        assert list(got[1]) == list(ref[1])
        assert got[2] == ref[2]


def test_graph_order_rejects_bad_input():
    L = _capi.load()
    e = np.array([[0, 5]], np.int32)
    w = np.array([1.0])
    order = np.zeros(2, np.int32)
    assert L.hsw_debug_graph_order(2, 1, e.ctypes.data, w.ctypes.data, 10, order.ctypes.data, None, None) == -7
    assert "out of range" in _capi.last_error()
