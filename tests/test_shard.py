"""CPU tests of the multi-GPU clique sharding.

The partitioner and the three-all-reduce algorithm are checked against the
single-process oracle, in-process and across two processes (gloo).
"""
import os

import numpy as np
import pytest

from helpers import rel
from oracle import hsde_oracle as O
from oracle import sharded_oracle as SO
from paper_1611_01828_b200.shard import gather_state, make_shards, scatter_state
from paper_1611_01828_b200.synthetic import block_arrow, make_config


@pytest.mark.parametrize("cfg,world", [(0, 2), (0, 3), (2, 4), (3, 2)])
def test_partition_invariants(cfg, world):
    cp = make_config(cfg)
    shards = make_shards(cp, world)
    ids = np.concatenate([s.clique_ids for s in shards])
    assert np.array_equal(ids, np.arange(cp.p))                     # contiguous, complete
    owned = np.zeros(cp.N_c, int)
    for s in shards:
        owned[s.covered[s.owned]] += 1
    assert np.all(owned == 1)                                        # one owner per coordinate
    slots = np.concatenate([s.slot_global for s in shards])
    assert np.array_equal(np.sort(slots), np.arange(cp.n_d))         # slots partitioned
    for s in shards:                                                 # local structure consistent
        lp = s.problem
        assert np.array_equal(lp.covered[lp.slot_cov], cp.covered[cp.slot_cov[s.slot_global]])
        assert np.array_equal(s.D, cp.D[s.covered])
        assert np.array_equal(s.covered[s.sep_local], np.flatnonzero(
            np.isin(np.arange(cp.N_c), s.covered))[np.isin(np.flatnonzero(
                np.isin(np.arange(cp.N_c), s.covered)), s.covered[s.sep_local])])
    rng = np.random.default_rng(0)
    u = rng.normal(size=cp.total)
    assert np.array_equal(gather_state(cp, shards, scatter_state(cp, shards, u)), u)


def test_block_arrow_separator_is_the_head():
    cp = make_config(0)
    shards = make_shards(cp, 4)
    assert shards[0].n_sep == 10 * 10  # h x h arrow head


def _oracle_run(cp, iters):
    st = {}

    def cb(k, p, d, g, tau, kap, u, w):
        st[k] = (u.copy(), (p, d, g))

    O.solve(cp, O.OracleSettings(max_iters=iters, tol=1e-300), callback=cb)
    return st


@pytest.mark.parametrize("cfg,world,iters", [(0, 2, 100), (0, 3, 60), (2, 3, 40)])
def test_sharded_algorithm_matches_single(cfg, world, iters):
    cp = make_config(cfg)
    shards = make_shards(cp, world)
    runs = [SO.ShardRun(s) for s in shards]
    logs = SO.drive_in_process([SO.rank_program(r, iters) for r in runs])
    u = gather_state(cp, shards, [r.u for r in runs])
    ref = _oracle_run(cp, iters)
    assert rel(u, ref[iters][0]) <= 1e-10
    for (k, p, d, g) in logs[0]:
        assert np.allclose((p, d, g), ref[k][1], rtol=1e-8)
    # every rank reports the same residuals
    assert all(l == logs[0] for l in logs)


def test_sharded_cta_cliques_four_ranks():
    cp = block_arrow(12, 24, 16, 50, 0.05, 7, "ctapath")
    shards = make_shards(cp, 4)
    runs = [SO.ShardRun(s) for s in shards]
    SO.drive_in_process([SO.rank_program(r, 40) for r in runs])
    u = gather_state(cp, shards, [r.u for r in runs])
    assert rel(u, _oracle_run(cp, 40)[40][0]) <= 1e-10


def _gloo_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cp = make_config(0)
    sh = make_shards(cp, world)[rank]
    run = SO.ShardRun(sh)
    log = SO.drive_torch_dist(SO.rank_program(run, 60))
    np.save(os.path.join(out_dir, f"u{rank}.npy"), run.u)
    np.save(os.path.join(out_dir, f"log{rank}.npy"), np.array(log))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gloo_two_processes(tmp_path):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    mp.spawn(_gloo_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    cp = make_config(0)
    shards = make_shards(cp, world)
    parts = [np.load(tmp_path / f"u{r}.npy") for r in range(world)]
    u = gather_state(cp, shards, parts)
    ref = _oracle_run(cp, 60)
    assert rel(u, ref[60][0]) <= 1e-10
    l0, l1 = np.load(tmp_path / "log0.npy"), np.load(tmp_path / "log1.npy")
    assert np.array_equal(l0, l1)
    assert np.allclose(l0[:, 1:], [ref[int(k)][1] for k in l0[:, 0]], rtol=1e-8)
