"""Pair sharding + record all-gather (dist.py) on 2 CPU ranks over gloo.

The GPU sweep is not available here, so each rank computes its shard with the
CPU oracle (test infrastructure) and the product's shard_range/gather_records
assemble the full record set, which must equal the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_03831_b200.dist import gather_records, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import oracle
    from paper_2405_03831_b200 import core, fnn, synth
    from paper_2405_03831_b200.grid import KnobGrid
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = fnn.load_weights(os.path.join(root, "tests", "golden", "weights.json"))
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    grid = KnobGrid([core.default_space(400.0), core.default_space(350.0)])
    P = n * (n - 1) // 2
    b, e = shard_range(P, rank, world)
    r = oracle.sweep(w, F, T, grid, b, e, threads=1)
    local = {"corun_grid_index": torch.from_numpy(r["corun_grid_index"].astype(np.int32)),
             "corun_time": torch.from_numpy(r["corun_time"]),
             "corun_chosen": torch.from_numpy(r["corun_chosen"].astype(np.uint8)),
             "weight": torch.from_numpy(r["weight"])}
    full = gather_records(local, P)
    if rank == 0:
        np.savez(out_path, **{k: v.numpy() for k, v in full.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for P in (0, 1, 7, 100, 32640):
        for world in (1, 2, 3, 8):
            spans = [shard_range(P, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gather_equals_single_process(tmp_path, weights):
    import sys
    import oracle
    from paper_2405_03831_b200 import core, synth
    from paper_2405_03831_b200.grid import KnobGrid
    n = 37                                  # odd pair count: unequal shards
    out = str(tmp_path / "full.npz")
    mp.start_processes(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    grid = KnobGrid([core.default_space(400.0), core.default_space(350.0)])
    ref = oracle.sweep(weights, F, T, grid, threads=1)
    assert np.array_equal(got["corun_grid_index"], ref["corun_grid_index"])
    assert np.array_equal(got["weight"], ref["weight"])
    assert np.array_equal(got["corun_chosen"].astype(bool), ref["corun_chosen"])
