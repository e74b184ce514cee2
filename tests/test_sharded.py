"""Direction-sharded source iteration: host logic and collectives.

CPU (gloo, world_size 2) with the oracle-backed test backend; GPU parity of the
device primitives against hsw_source_iteration in test_sharded_gpu below.
"""
import os
import sys
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_11080_b200 import problem as pb
from paper_1810_11080_b200.sharded import block_of, sharded_source_iteration

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _oracle_shard_backend import OracleShardBackend  # noqa: E402

PROB = dict(name="c1", cells=3, n_mu=2, n_az=4)   # 9 elements, 8 ordinates, Q2


def _problem():
    kw = dict(PROB)
    return pb.config(kw.pop("name"), **kw)


def test_blocks_partition_the_ordinates():
    for nd in (1, 7, 8, 256):
        for world in range(1, min(nd, 9) + 1):
            blocks = [block_of(nd, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == nd
            assert all(b[0] == a[1] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        block_of(4, 0, 5)
    with pytest.raises(ValueError):
        block_of(4, 4, 4)


def test_one_rank_reproduces_the_oracle_source_iteration():
    prob = _problem()
    be = OracleShardBackend(prob)
    res = sharded_source_iteration(be, tolerance=1e-10, max_iterations=200, criterion="phi_rel_l2",
                                   return_psi=True)
    ref = be.o.source_iteration(1e-10, 200, 1)
    assert res.converged and ref["converged"]
    assert res.iterations == ref["iterations"]
    assert np.array_equal(res.phi, ref["phi"])
    assert np.array_equal(res.psi, ref["psi"])
    assert res.errors == list(ref["error"]) and res.phi_rels == list(ref["phi_rel"])


def test_local_blocks_are_bit_identical_to_one_block():
    prob = _problem()
    one = sharded_source_iteration(OracleShardBackend(prob), tolerance=1e-9, criterion="psi_linf",
                                   return_psi=True)
    three = sharded_source_iteration(OracleShardBackend(prob), tolerance=1e-9, criterion="psi_linf",
                                     local_blocks=3, return_psi=True)
    assert three.blocks == [(0, 2), (2, 5), (5, 8)]
    assert one.iterations == three.iterations
    assert np.array_equal(one.phi, three.phi) and np.array_equal(one.psi, three.psi)
    assert one.errors == three.errors


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = sharded_source_iteration(OracleShardBackend(_problem()), tolerance=1e-10, max_iterations=200,
                                       criterion="phi_rel_l2", return_psi=True)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), phi=res.phi, psi=res.psi, blocks=np.array(res.blocks),
                 it=res.iterations, conv=res.converged, errs=np.array(res.errors), rels=np.array(res.phi_rels))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_match_one_rank_bit_for_bit(world):
    prob = _problem()
    ref = sharded_source_iteration(OracleShardBackend(prob), tolerance=1e-10, max_iterations=200,
                                   criterion="phi_rel_l2", return_psi=True)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), tmp), nprocs=world, join=True)
        outs = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
    psi = np.concatenate([o["psi"] for o in outs])
    for r, o in enumerate(outs):
        assert tuple(o["blocks"][0]) == block_of(prob.num_ordinates, r, world)
        assert int(o["it"]) == ref.iterations and bool(o["conv"])
        assert np.array_equal(o["phi"], ref.phi)            # chained prefix: identical bits on every rank
        assert list(o["errs"]) == ref.errors and list(o["rels"]) == ref.phi_rels
    assert np.array_equal(psi, ref.psi)


@pytest.mark.gpu
def test_device_shards_match_hsw_source_iteration_bit_for_bit():
    """The hsw_shard_* primitives (range worklists, chained FMA phi, norm tree)
    reproduce the single-device source iteration exactly, for 1 and 4 blocks."""
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200.sharded import DeviceShardBackend
    for name, kw in (("c1", {}), ("c3", dict(cells=4, n_mu=2, n_az=4))):
        prob = pb.config(name, **kw)
        s = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-8, criterion="phi_rel_l2"))
        state, hist = s.source_iteration()
        for blocks in (None, 4):
            res = sharded_source_iteration(DeviceShardBackend(s), tolerance=1e-8, criterion="phi_rel_l2",
                                           local_blocks=blocks, return_psi=True)
            assert res.converged and hist.converged
            assert res.iterations == hist.iterations()
            assert np.array_equal(res.phi, state.phi)
            assert np.array_equal(res.psi, state.psi)
            assert res.errors == list(hist.error) and res.phi_rels == list(hist.phi_rel)


@pytest.mark.gpu
def test_shard_sweep_host_matches_the_all_ordinate_sweep():
    """hsw_shard_sweep_host (a rank's ordinate block end to end with host buffers,
    H2D / sweep / D2H pipelined over sub-blocks) equals rows [d0, d1) of the
    all-ordinate host-pointer sweep, bit for bit, at a size where the pipeline runs."""
    import ctypes as C
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200 import _capi
    prob = pb.config("c4", cells=16, n_mu=4, n_az=16)   # 4096 hexes, 64 ordinates: 134 MB of psi
    s = pk.SweepSolver(prob)
    L = _capi.load()
    rng = np.random.default_rng(5)
    N, nd = prob.num_dofs, prob.num_ordinates
    phi = rng.uniform(0, 1, N)
    psi_old = rng.uniform(-0.5, 1.0, (nd, N))
    ref = s.sweep(-1, phi, psi_old)
    # an independent path: per-ordinate sweeps (per-level launches, no sub-block pipeline)
    for d in (0, 17, 39, 40, 63):
        assert np.array_equal(s.sweep(d, phi, psi_old[d]), ref[d]), d
    for d0, d1 in ((0, nd), (16, 48), (40, 64)):
        blk_old = np.ascontiguousarray(psi_old[d0:d1])
        blk_new = np.empty_like(blk_old)
        rc = L.hsw_shard_sweep_host(s.handle, d0, d1, C.c_void_p(phi.ctypes.data), C.c_void_p(blk_old.ctypes.data),
                                    C.c_void_p(blk_new.ctypes.data))
        assert rc == 0, _capi.last_error()
        assert np.array_equal(blk_new, ref[d0:d1]), (d0, d1)
        # launches summed over the pipelined sub-blocks: scatter + one dataflow launch each
        assert L.hsw_last_launch_count(s.handle) >= 2


def test_shard_handle_plan_equals_the_full_plan():
    """hsw_problem_desc::ordinate_begin/end (a rank's shard): the shard's orders / cut
    sets equal the full handle's, other ordinates and all-ordinate calls are refused."""
    import paper_1810_11080_b200 as pk
    prob = pb.config("c3", cells=3, n_mu=2, n_az=4)
    full = pk.SweepSolver(prob, device=-1)
    part = pk.SweepSolver(prob, device=-1, ordinate_range=(2, 6))
    assert part.ordinate_range == (2, 6)
    for d in range(2, 6):
        a, b = full.ordering(d), part.ordering(d)
        assert (a.order == b.order).all() and (a.lagged_edges == b.lagged_edges).all() and (a.level == b.level).all()
    assert part.total_lagged_edges() == sum(len(full.ordering(d).lagged_edges) for d in range(2, 6))
    with pytest.raises(IndexError, match="shard"):
        part.ordering(1)
    with pytest.raises(IndexError):
        pk.SweepSolver(prob, device=-1, ordinate_range=(5, 3))


@pytest.mark.gpu
def test_shard_handles_reproduce_the_full_handle_bit_for_bit():
    """Two shard handles (what two ranks create) sweep their blocks and chain phi exactly
    like one full handle's blocks: psi and phi identical bits for three iterations."""
    import torch
    import paper_1810_11080_b200 as pk
    from paper_1810_11080_b200.sharded import DeviceShardBackend
    prob = pb.config("c4", cells=6, n_mu=2, n_az=8)
    nd = prob.num_ordinates
    blocks = [(0, 7), (7, nd)]
    full = DeviceShardBackend(pk.SweepSolver(prob))
    parts = [DeviceShardBackend(pk.SweepSolver(prob, ordinate_range=b)) for b in blocks]
    for be in [full] + parts:
        be.reset()
    phi_f = full.zeros()
    phi_p = parts[0].zeros()
    for it in range(3):
        for (d0, d1) in blocks:
            full.sweep(d0, d1, phi_f)
        for be, (d0, d1) in zip(parts, blocks):
            be.sweep(d0, d1, phi_p)
        pf = None
        for (d0, d1) in blocks:
            out = full.zeros()
            full.phi_partial(d0, d1, pf, out)
            pf = out
        pp = None
        for be, (d0, d1) in zip(parts, blocks):
            out = be.zeros()
            be.phi_partial(d0, d1, pp, out)
            pp = out
        assert torch.equal(pf, pp), it
        for be, (d0, d1) in zip(parts, blocks):
            assert np.array_equal(be.psi(d0, d1), full.psi(d0, d1)), (it, d0)
        full.advance(pf)
        for be in parts:
            be.advance(pp)
        phi_f, phi_p = pf, pp
    with pytest.raises(IndexError):
        parts[0].solver.source_iteration()
