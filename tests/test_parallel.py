"""CPU, world_size 2 over gloo: the multi-GPU host logic.

* partitions: chains exactly as kreg_register_sequence_chains, row shards;
* the collective callback (TorchCollective) through its C function pointer;
* a row-sharded registration (C4) through the product solver with the C
  oracle standing in for the device (tests/native/mock_round.cpp): two ranks,
  each with half of the source rows, combined every round through gloo, must
  reproduce the unsharded registration.
"""
import ctypes as C
import math
import os
import socket
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2012_03683_b200 import _abi, parallel, synth
from paper_2012_03683_b200.types import Isometry, KernelParams, PointCloud, RegistrationConfig, RegistrationResult
from paper_2012_03683_b200.types import compose, inverse

HERE = os.path.dirname(os.path.abspath(__file__))
MOCK = os.path.join(HERE, "native", "libmock_solver.so")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(fn, args=(world, port) + args, nprocs=world, join=True)


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ----------------------------------------------------------- partitions
def test_chain_spans_match_engine_partition():
    for n_frames, n_chains in [(2, 1), (9, 3), (4097, 64), (10, 20), (33, 8)]:
        spans = parallel.chain_spans(n_frames, n_chains)
        m = n_frames - 1
        nc = min(n_chains, m)
        assert spans == [(m * c // nc, m * (c + 1) // nc) for c in range(nc)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
            assert e0 == b1 and b0 < e0
        for world in (1, 2, 3, 8):
            got = [s for r in range(world) for s in parallel.rank_spans(spans, r, world)]
            assert got == spans
    with pytest.raises(ValueError):
        parallel.chain_spans(1, 1)


def test_row_shards_partition_the_source():
    X, Z, _ = synth.kitti_pair(3, 2000)
    for world in (1, 2, 3, 8):
        parts = [parallel.shard_rows(Z, r, world) for r in range(world)]
        assert sum(p.size() for p in parts) == Z.size()
        got = np.concatenate([p.positions for p in parts])
        assert np.array_equal(np.sort(got.view("f8,f8,f8"), axis=0), np.sort(Z.positions.copy().view("f8,f8,f8"), axis=0))
        # Morton-contiguous shards are spatially compact: bbox volume well below the full cloud's
        if world == 2:
            vol = lambda P: np.prod(P.max(0) - P.min(0))  # noqa: E731
            assert max(vol(p.positions) for p in parts) < vol(Z.positions)
    with pytest.raises(ValueError):
        parallel.shard_rows(PointCloud(Z.positions[:1]), 0, 2)


def test_assemble_sequence_composes_trajectory():
    rng = synth.SplitMix64(4)
    rel = [synth.random_isometry(rng, 0.1, 0.2) for _ in range(5)]
    parts = [[(p, rel[p].as12().tolist(), 0, 1, 0.5, 10 + p) for p in (0, 1, 2)],
             [(p, rel[p].as12().tolist(), int(p == 4), 1, 0.5, 10 + p) for p in (3, 4)]]
    seq = parallel.assemble_sequence(6, parts)
    T = Isometry()
    for k in range(5):
        T = compose(T, rel[k])
        assert np.allclose(seq.trajectory[k + 1].as12(), T.as12(), atol=1e-14)
    assert list(seq.fallback) == [0, 0, 0, 0, 1] and list(seq.iterations) == [10, 11, 12, 13, 14]


# ------------------------------------------------------------ collective
def _collective_worker(rank, world, port, out_dir):
    _init(rank, world, port)
    rows = []
    for det in (True, False):  # all_gather + rank-order sum, and the two all_reduces
        coll = parallel.TorchCollective(deterministic=det)
        sums = (C.c_double * 3)(1.0 + rank, 10.0 * rank, -2.0)
        maxes = (C.c_double * 2)(float(rank), 5.0 - rank)
        rc = coll.c_fn(None, sums, 3, maxes, 2)
        rows.append([rc, *sums, *maxes])
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(rows, dtype=np.float64))
    assert parallel.reduce_scalar(float(rank + 1), "max") == float(world)
    assert parallel.reduce_scalar(1.0, "sum") == float(world)


def test_collective_callback_over_gloo():
    with tempfile.TemporaryDirectory() as d:
        _spawn(_collective_worker, 2, d)
        for r in range(2):
            for v in np.load(os.path.join(d, f"r{r}.npy")):
                assert v[0] == 0
                assert np.array_equal(v[1:4], [3.0, 10.0, -4.0])
                assert np.array_equal(v[4:6], [1.0, 5.0])


# ------------------------------------- row-sharded registration (mock device)
def _mock():
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "native")], stderr=subprocess.DEVNULL)
    L = C.CDLL(MOCK)
    L.mock_register_rows.argtypes = [C.POINTER(_abi.kreg_cloud_view), C.POINTER(_abi.kreg_cloud_view), _abi.dptr,
                                     C.POINTER(_abi.kreg_kernel_params), C.POINTER(_abi.kreg_registration_config),
                                     C.POINTER(_abi.kreg_registration_result), C.c_int, C.c_longlong,
                                     parallel_fn_type(), C.c_void_p]
    return L


def parallel_fn_type():
    from paper_2012_03683_b200 import api
    return api.COLLECTIVE_FN


def _case():
    X = synth.make_box_cloud(41, 400, False)
    rng = synth.SplitMix64(42)
    Z = PointCloud(inverse(synth.se3_exp(synth.random_twist(rng, 6.0 * math.pi / 180.0, 0.03))).apply(X.positions))
    cfg = RegistrationConfig(init_lengthscale=0.15, min_lengthscale=0.07, subsequent_lengthscale=0.15,
                             stabilization_window=3, max_iterations=300)
    return X, Z, Isometry(), KernelParams(), cfg


def _run(L, X, Zr, n_total, init, p, cfg, coll):
    buf = _abi.TraceBuffers(cfg.max_iterations)
    t = init.as12()
    c = cfg.cstruct()
    fn = coll.c_fn if coll is not None else parallel_fn_type()()
    rc = L.mock_register_rows(X.view(), Zr.view(), _abi.as_ptr(t), p.cstruct(), C.byref(c), C.byref(buf.struct), 2,
                              n_total, fn, None)
    return rc, RegistrationResult.from_buffers(buf)


def _sharded_worker(rank, world, port, out_dir):
    _init(rank, world, port)
    L = _mock()
    X, Z, init, p, cfg = _case()
    Zr = parallel.shard_rows(Z, rank, world)
    coll = parallel.TorchCollective()
    rc, res = _run(L, X, Zr, Z.size(), init, p, cfg, coll)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), rc=rc, T=res.transform.as12(), obj=res.objective_trace,
             it=res.iterations, pc=res.pair_count_trace, calls=coll.calls)


def test_row_sharded_registration_matches_unsharded():
    L = _mock()
    X, Z, init, p, cfg = _case()
    rc, want = _run(L, X, Z, Z.size(), init, p, cfg, None)
    assert rc == 0 and want.iterations > 10
    with tempfile.TemporaryDirectory() as d:
        _spawn(_sharded_worker, 2, d)
        got = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    for g in got:
        assert int(g["rc"]) == 0
        assert int(g["calls"]) > 0
        # ranks agree exactly (identical reduced values -> identical decisions)
        assert np.array_equal(g["T"], got[0]["T"]) and np.array_equal(g["obj"], got[0]["obj"])
        # and match the unsharded registration (sums only re-associated)
        assert int(g["it"]) == want.iterations
        assert np.array_equal(g["pc"], want.pair_count_trace)
        assert np.allclose(g["obj"], want.objective_trace, rtol=1e-11, atol=0)
        assert np.allclose(g["T"], want.transform.as12(), rtol=0, atol=1e-9)
