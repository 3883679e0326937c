"""The sharded multi-rank sweep (dist.ShardedSweep) on one GPU: 2 and 3 ranks share
cuda:0 over gloo (this environment has one GPU; on 8 GPUs the same code runs one
rank per GPU over NCCL).  The 11-byte wire records gathered to rank 0 and
rank 0's device rebuild (cs_unpack_gathered) must give exactly the
single-process graph, and the rebuilt records must equal the fp64 oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    from paper_2405_03831_b200 import core, fnn, synth
    from paper_2405_03831_b200.device import to_device_inputs
    from paper_2405_03831_b200.dist import ShardedSweep
    from paper_2405_03831_b200.grid import KnobGrid
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = fnn.load_weights(os.path.join(root, "tests", "golden", "weights.json"))
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    grid = KnobGrid([core.default_space(400.0), core.default_space(350.0)])
    sh = ShardedSweep(w, grid, n, device=torch.device("cuda", 0))
    d_f, d_b = to_device_inputs(F, T, sh.plan.device)
    sh.run_checked(d_f, d_b)
    M = sh.matrix
    torch.cuda.synchronize()
    rec = sh.records()
    assert (rank == 0) == (rec is not None) == (M is not None)
    if rank == 0:
        np.savez(out_path, matrix=M.cpu().numpy(), **{k: v.cpu().numpy() for k, v in rec.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_rebuilds_the_graph(tmp_path, weights, world):
    import oracle
    from conftest import workload
    from paper_2405_03831_b200 import core
    from paper_2405_03831_b200.grid import KnobGrid
    from paper_2405_03831_b200.sweep import sweep_pairs
    from paper_2405_03831_b200 import synth
    n = 150
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(world, _free_port(), n, out), nprocs=world,
                       start_method="spawn", join=True)
    got = dict(np.load(out))
    spaces = [core.default_space(400.0), core.default_space(350.0)]
    single = sweep_pairs(weights, synth.generate_jobs(0, synth.mixed_archetypes(n)), spaces)
    assert np.array_equal(got["matrix"], single.matrix)
    F, T = workload(n)
    ref = oracle.sweep(weights, F, T, KnobGrid(spaces))
    for l in range(2):
        assert np.array_equal(got["corun_grid_index"][l], ref["corun_grid_index"][l])
        assert np.array_equal(got["weight"][l], ref["weight"][l])
        assert np.array_equal(got["corun_chosen"][l].astype(bool), ref["corun_chosen"][l])
        assert np.array_equal(got["corun_time"][l], ref["corun_time"][l])
