"""The multi-rank exchange of dist.py on 2 and 3 CPU ranks over gloo.

No GPU here, so each rank computes its pair shard with the CPU oracle (test
infrastructure) and packs it into the 11-byte wire format with a numpy
mirror of cs_pack_records; the PRODUCT's shard_range / shard_cap /
wire_layout / gather_to_root move the buffers to rank 0, which rebuilds the
full record set (numpy mirror of cs_unpack_gathered: weight re-derived from
the solo times) -- it must equal the single-process oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_03831_b200.dist import gather_to_root, shard_cap, shard_range, wire_layout


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pack(r, L, P, cap):
    lay = wire_layout(cap, L)
    buf = np.zeros(lay["total"], dtype=np.uint8)
    t = buf[lay["corun_time"]:].view(np.float64)[:L * cap].reshape(L, cap)
    ix = buf[lay["corun_grid_index"]:lay["corun_chosen"]].view(np.uint16)[:L * cap].reshape(L, cap)
    fl = buf[lay["corun_chosen"]:][:L * cap].reshape(L, cap)
    t[:, :P] = r["corun_time"][:, :P]
    g = r["corun_grid_index"][:, :P]
    ix[:, :P] = np.where(g < 0, 0xFFFF, g).astype(np.uint16)
    fl[:, :P] = r["corun_chosen"][:, :P]
    return buf


def _unpack(blocks, world, P, n, L, cap, solo_time):
    lay = wire_layout(cap, L)
    out = {k: np.empty((L, P), dtype=d) for k, d in (
        ("corun_grid_index", np.int32), ("corun_time", np.float64), ("corun_chosen", bool),
        ("weight", np.float64))}
    iu, ju = np.triu_indices(n, 1)
    for r in range(world):
        b, e = shard_range(P, r, world)
        buf = blocks[r]
        t = buf[lay["corun_time"]:].view(np.float64)[:L * cap].reshape(L, cap)[:, :e - b]
        ix = buf[lay["corun_grid_index"]:lay["corun_chosen"]].view(np.uint16)[:L * cap].reshape(L, cap)[:, :e - b]
        fl = buf[lay["corun_chosen"]:][:L * cap].reshape(L, cap)[:, :e - b].astype(bool)
        out["corun_time"][:, b:e] = t
        out["corun_grid_index"][:, b:e] = np.where(ix == 0xFFFF, -1, ix.astype(np.int32))
        out["corun_chosen"][:, b:e] = fl
        for l in range(L):
            st = solo_time[l]
            solo = (0.0 + st[iu[b:e]]) + st[ju[b:e]]
            out["weight"][l, b:e] = np.where(fl[l], t[l], solo)
    return out


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
    P, L = n * (n - 1) // 2, grid.n_budgets
    b, e = shard_range(P, rank, world)
    cap = shard_cap(P, world)
    r = oracle.sweep(w, F, T, grid, b, e, threads=1)
    wire = torch.from_numpy(_pack(r, L, e - b, cap))
    got = gather_to_root(wire)
    assert (got is not None) == (rank == 0)
    if rank == 0:
        full = _unpack([got[k].numpy() for k in range(world)], world, P, n, L, cap, r["solo_time"])
        np.savez(out_path, **full)
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
            assert max(sizes) == shard_cap(P, world)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_wire_layout_matches_the_abi():
    """The Python mirror of the wire layout agrees with cs_wire_records_bytes."""
    from paper_2405_03831_b200 import _native as nat
    lib = nat.sweep_lib()
    for cap, L in ((1, 1), (1000, 2), (4_193_280, 1), (52_378, 5)):
        assert wire_layout(cap, L)["total"] == lib.cs_wire_records_bytes(cap, L)
        assert lib.cs_wire_records_bytes(cap, L) < 11 * cap * L + 3 * 256


@pytest.mark.parametrize("world", [2, 3])
def test_gather_to_root_rebuilds_the_oracle_records(tmp_path, weights, world):
    import oracle
    from paper_2405_03831_b200 import core, synth
    from paper_2405_03831_b200.grid import KnobGrid
    n = 37                                  # odd pair count: unequal shards
    out = str(tmp_path / "full.npz")
    mp.start_processes(_worker, args=(world, _free_port(), n, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    grid = KnobGrid([core.default_space(400.0), core.default_space(350.0)])
    ref = oracle.sweep(weights, F, T, grid, threads=1)
    for k in ("corun_grid_index", "corun_time", "weight"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["corun_chosen"], ref["corun_chosen"])
