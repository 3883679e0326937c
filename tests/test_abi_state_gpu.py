"""State kept between host-ABI calls, and concurrent callers.

* cs_build_graph_host keeps uploads resident only in a workspace the caller
  retained (cs_workspace_retain); a released or never-retained workspace is
  uploaded into on every call, so memory reused at the same address -- even
  poisoned with 0xFF -- gives exact results.
* The Python entry points share cached SweepPlans; concurrent callers must
  see exactly the serial results (the reference promises thread-safe pure
  functions, core.py:3-6, scheduler.py:56-71).
"""

import ctypes
import threading

import numpy as np
import pytest
import torch

import oracle
from conftest import workload
import paper_2405_03831_b200 as cs
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import NetworkABI
from paper_2405_03831_b200.grid import KnobGrid
from paper_2405_03831_b200.host_abi import _host_grid

pytestmark = pytest.mark.gpu


def _call(lib, net, cgrid, F, T, ws_ptr, ws_bytes, L, stream=None):
    n = len(T)
    W = np.zeros((L, n, n))
    st = np.empty((L, n))
    ss = np.empty((L, n), np.int32)
    cl = np.zeros(L, np.uint64)
    rc = lib.cs_build_graph_host(net.ref(), ctypes.byref(cgrid), nat.ptr(F), nat.ptr(T), n, 1e-5,
                                 ws_ptr, ws_bytes, nat.ptr(W), nat.CsPairOut(),
                                 nat.CsSoloOut(nat.ptr(st), nat.ptr(ss, nat.c_int32_p), None),
                                 cl.ctypes.data_as(nat.c_ull_p), stream)
    nat.check(rc, "cs_build_graph_host")
    return W, st, ss


def _expected(weights, F, T, grid, n):
    ref = oracle.sweep(weights, F, T, grid)
    iu, ju = np.triu_indices(n, 1)
    return iu, ju, ref


def test_reused_and_poisoned_workspace_is_exact(weights):
    lib = nat.sweep_lib()
    n = 96
    F, T = workload(n, 3)
    grid = KnobGrid([core.default_space(400.0)])
    cgrid, keep = _host_grid(grid)
    net = NetworkABI(weights)
    nbytes = lib.cs_build_graph_workspace_bytes(n, ctypes.byref(cgrid))
    iu, ju, ref = _expected(weights, F, T, grid, n)

    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    ptr = (ws.data_ptr() + 255) & ~255
    nat.check(lib.cs_workspace_retain(ptr, nbytes), "retain")
    for _ in range(3):                      # fresh, cached, cached
        W, _, _ = _call(lib, net, cgrid, F, T, ptr, nbytes, 1)
        assert np.array_equal(W[0][iu, ju], ref["weight"][0])
    nat.check(lib.cs_workspace_release(ptr), "release")
    del ws
    torch.cuda.synchronize()

    ws2 = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    ptr2 = (ws2.data_ptr() + 255) & ~255
    ws2.fill_(0xFF)                         # NaN everywhere: nothing may survive
    torch.cuda.synchronize()
    W, _, _ = _call(lib, net, cgrid, F, T, ptr2, nbytes, 1)   # never retained
    assert np.array_equal(W[0][iu, ju], ref["weight"][0])
    assert np.all(np.diag(W[0]) == 0.0)
    # retained after the poison: its first call uploads everything
    ws2.fill_(0xFF)
    torch.cuda.synchronize()
    nat.check(lib.cs_workspace_retain(ptr2, nbytes), "retain")
    W, _, _ = _call(lib, net, cgrid, F, T, ptr2, nbytes, 1)
    assert np.array_equal(W[0][iu, ju], ref["weight"][0])
    assert np.all(np.diag(W[0]) == 0.0)
    nat.check(lib.cs_workspace_release(ptr2), "release")


def test_device_alloc_free_realloc_is_exact(weights):
    """cs_device_free drops the retained state: a new allocation at the same
    address starts from nothing."""
    lib = nat.sweep_lib()
    n = 64
    F, T = workload(n, 4)
    grid = KnobGrid([core.default_space(350.0)])
    cgrid, keep = _host_grid(grid)
    net = NetworkABI(weights)
    nbytes = lib.cs_build_graph_workspace_bytes(n, ctypes.byref(cgrid))
    iu, ju, ref = _expected(weights, F, T, grid, n)
    for _ in range(3):
        p = ctypes.c_void_p()
        nat.check(lib.cs_device_alloc(nbytes, ctypes.byref(p)), "alloc")
        nat.check(lib.cs_workspace_retain(p, nbytes), "retain")
        W, _, _ = _call(lib, net, cgrid, F, T, p, nbytes, 1)
        assert np.array_equal(W[0][iu, ju], ref["weight"][0])
        nat.check(lib.cs_device_free(p), "free")


def test_retained_workspace_follows_network_changes(weights):
    lib = nat.sweep_lib()
    n = 48
    F, T = workload(n, 6)
    grid = KnobGrid([core.default_space(400.0)])
    cgrid, keep = _host_grid(grid)
    other = fnn.initialize_weights(11, weights.feature_bounds)
    nbytes = lib.cs_build_graph_workspace_bytes(n, ctypes.byref(cgrid))
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    ptr = (ws.data_ptr() + 255) & ~255
    nat.check(lib.cs_workspace_retain(ptr, nbytes), "retain")
    stream = torch.cuda.Stream()
    try:
        for w in (weights, other, weights, weights, other):
            net = NetworkABI(w)
            iu, ju, ref = _expected(w, F, T, grid, n)
            with torch.cuda.stream(stream):
                W, _, _ = _call(lib, net, cgrid, F, T, ptr, nbytes, 1, stream.cuda_stream)
            assert np.array_equal(W[0][iu, ju], ref["weight"][0])
    finally:
        lib.cs_workspace_release(ptr)


def test_concurrent_decide_pair_equals_serial(weights):
    jobs = synth.generate_jobs(7, synth.mixed_archetypes(40))
    space = core.default_space(400.0)
    pairs = [(i, j) for i in range(0, 40, 3) for j in range(i + 1, 40, 5)]
    serial = [cs.decide_pair(weights, jobs[i], jobs[j], space) for i, j in pairs]
    results = [None] * len(pairs)
    errors = []

    def worker(k0):
        try:
            for k in range(k0, len(pairs), 8):
                i, j = pairs[k]
                results[k] = cs.decide_pair(weights, jobs[i], jobs[j], space)
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert results == serial
    # build_graph from several threads at once (shared cached plan)
    inp = cs.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=40), weights)
    ref = cs.build_graph(inp).weights
    outs = [None] * 4

    def bg(k):
        outs[k] = cs.build_graph(inp).weights

    threads = [threading.Thread(target=bg, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for o in outs:
        assert np.array_equal(o, ref)


def test_chunked_host_call_overlaps_copies_and_stays_exact(weights):
    """~18 MB of pinned D2H (n = 1,100, one budget, records): cs_build_graph_host sweeps
    in row chunks and copies each finished row block + its records on a second
    stream while the next chunk computes.  Eager, captured and replayed calls
    (on a non-default stream) all equal the fp64 oracle bit for bit."""
    from paper_2405_03831_b200.host_abi import HostGraphCall
    n = 1100
    F, T = workload(n, 11)
    grid = KnobGrid([core.default_space(375.0)])
    ref = oracle.sweep(weights, F, T, grid)
    iu, ju = np.triu_indices(n, 1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        call = HostGraphCall(weights, grid, n, with_records=True)
        try:
            for _ in range(4):                 # eager, eager, capture, replay
                call.h_weights[...] = -1.0
                call.h_idx[...] = -7
                out = call(F, T)
                W = out["weights"][0]
                assert np.array_equal(W[iu, ju], ref["weight"][0])
                assert np.array_equal(W[ju, iu], ref["weight"][0])
                assert np.array_equal(call.h_idx[0], ref["corun_grid_index"][0])
                assert np.array_equal(call.h_ct[0], ref["corun_time"][0])
                assert np.array_equal(call.h_ch[0].astype(bool), ref["corun_chosen"][0])
                assert np.array_equal(call.h_solo_time[0], ref["solo_time"][0])
        finally:
            call.close()


def test_zero_copy_epilogue_with_misaligned_pinned_outputs(weights):
    """Every destination pinned but the record arrays placed at odd offsets
    inside one pinned buffer: the one-kernel epilogue (16-byte stores where
    both ends are aligned, bytewise otherwise) still delivers every output
    exactly; repeated calls on a non-default stream replay a captured graph."""
    lib = nat.sweep_lib()
    n = 130
    F, T = workload(n, 5)
    grid = KnobGrid([core.default_space(400.0)])
    cgrid, keep = _host_grid(grid)
    net = NetworkABI(weights)
    P = n * (n - 1) // 2
    nbytes = lib.cs_build_graph_workspace_bytes(n, ctypes.byref(cgrid))
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    ws_ptr = (ws.data_ptr() + 255) & ~255
    nat.check(lib.cs_workspace_retain(ws_ptr, nbytes), "retain")
    iu, ju, ref = _expected(weights, F, T, grid, n)
    pin = lambda nb: torch.empty(nb, dtype=torch.uint8, pin_memory=True).numpy()
    raw = pin(8 * P + 4 * P + P + 64)
    idx = raw[1:1 + 4 * P].view(np.int32)            # odd offsets: bytewise path
    ct = raw[4 * P + 3:4 * P + 3 + 8 * P].view(np.float64)
    ch = raw[12 * P + 5:12 * P + 5 + P]
    hf = pin(F.nbytes).view(np.float64).reshape(F.shape); hf[...] = F
    hb = pin(T.nbytes).view(np.float64); hb[...] = T
    W = pin(8 * n * n).view(np.float64).reshape(1, n, n)
    st = pin(8 * n).view(np.float64)
    ss = pin(4 * n).view(np.int32)
    cl = pin(8).view(np.uint64)
    s = torch.cuda.Stream()
    try:
        for _ in range(4):                       # eager, eager, capture, replay
            W[...] = -1.0; idx[...] = -9; ct[...] = 0.0; ch[...] = 7
            rc = lib.cs_build_graph_host(net.ref(), ctypes.byref(cgrid), nat.ptr(hf), nat.ptr(hb), n,
                                         1e-5, ws_ptr, nbytes, nat.ptr(W),
                                         nat.CsPairOut(nat.ptr(idx, nat.c_int32_p), nat.ptr(ct),
                                                       nat.ptr(ch, nat.c_uint8_p), None),
                                         nat.CsSoloOut(nat.ptr(st), nat.ptr(ss, nat.c_int32_p), None),
                                         cl.ctypes.data_as(nat.c_ull_p), s.cuda_stream)
            nat.check(rc, "cs_build_graph_host")
            assert np.array_equal(W[0][iu, ju], ref["weight"][0])
            assert np.array_equal(W[0][ju, iu], ref["weight"][0])
            assert np.array_equal(idx, ref["corun_grid_index"][0])
            assert np.array_equal(ct, ref["corun_time"][0])
            assert np.array_equal(ch.astype(bool), ref["corun_chosen"][0])
            assert np.array_equal(st, ref["solo_time"][0])
    finally:
        lib.cs_workspace_release(ws_ptr)


def test_chunked_host_call_with_two_budgets(weights):
    """Two budgets, ~17 MB of pinned outputs: the row-chunked call keeps each
    chunk's records budget-major in its own workspace slice and copies them to
    their places in the L x P host arrays; every budget equals the oracle."""
    from paper_2405_03831_b200.host_abi import HostGraphCall
    n = 760
    F, T = workload(n, 13)
    grid = KnobGrid([core.default_space(400.0), core.default_space(350.0)])
    ref = oracle.sweep(weights, F, T, grid)
    iu, ju = np.triu_indices(n, 1)
    call = HostGraphCall(weights, grid, n, with_records=True)
    try:
        for _ in range(3):
            call.h_weights[...] = -1.0
            call.h_idx[...] = -7
            out = call(F, T)
            for l in range(2):
                W = out["weights"][l]
                assert np.array_equal(W[iu, ju], ref["weight"][l])
                assert np.array_equal(W[ju, iu], ref["weight"][l])
                assert np.array_equal(call.h_idx[l], ref["corun_grid_index"][l])
                assert np.array_equal(call.h_ct[l], ref["corun_time"][l])
                assert np.array_equal(call.h_ch[l].astype(bool), ref["corun_chosen"][l])
                assert np.array_equal(call.h_solo_time[l], ref["solo_time"][l])
            assert int(call.h_clamps[0]) >= 0
    finally:
        call.close()


def test_overlapped_small_call_two_budgets(weights):
    """Below the chunking threshold with every destination pinned: the bulk
    copy of matrix + records runs beside k_resolve and k_call_fixup re-copies
    the resolved pairs.  Two budgets and a wide ambiguity band (rel_eps
    2e-3: thousands of pairs go through k_resolve and the fixup); eager,
    captured and replayed calls equal the oracle."""
    from paper_2405_03831_b200.host_abi import HostGraphCall
    n = 200
    F, T = workload(n, 17)
    grid = KnobGrid([core.default_space(400.0), core.default_space(375.0)])
    ref = oracle.sweep(weights, F, T, grid)
    iu, ju = np.triu_indices(n, 1)
    call = HostGraphCall(weights, grid, n, with_records=True, rel_eps=2e-3)
    try:
        for _ in range(4):
            call.h_weights[...] = -1.0
            call.h_idx[...] = -7
            call.h_ct[...] = 0.0
            out = call(F, T)
            for l in range(2):
                W = out["weights"][l]
                assert np.array_equal(W[iu, ju], ref["weight"][l])
                assert np.array_equal(W[ju, iu], ref["weight"][l])
                assert np.array_equal(call.h_idx[l], ref["corun_grid_index"][l])
                assert np.array_equal(call.h_ct[l], ref["corun_time"][l])
                assert np.array_equal(call.h_ch[l].astype(bool), ref["corun_chosen"][l])
                assert np.array_equal(call.h_solo_split[l], ref["solo_split"][l])
    finally:
        call.close()
