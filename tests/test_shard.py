"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 path: unit
sharding and the end-of-run record gather (the only collective).  The
tracking itself is per-GPU; here each rank produces its records with the
oracle so the test runs without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_00463_b200.shard import gather_bytes, shard_list, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 5, 12, 32, 512):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                rr = shard_range(n, world, r)
                seen.extend(rr)
                assert len(rr) in (n // world, n // world + 1)
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1907_00463_b200 import abi
        # config-2-like channel batch sharding: 6 channels over the ranks
        fs = 2.048e6
        rng = np.random.default_rng(0)  # same stream on every rank
        x = (rng.uniform(-1, 1, 2048 * 12) + 1j * rng.uniform(-1, 1, 2048 * 12))
        chans = [oracle.init_channel(p, 100.0 * p, 0, 37 * p, 0, fs) for p in range(1, 7)]
        mine = shard_list(list(range(6)), world, rank)
        recs = []
        for c in mine:
            _, done, r, _ = oracle.track_run([chans[c]], [0], [x], 2048, abi.TrackingCfg.default(),
                                             abi.Taps.epl(0.5), fs, 8)
            recs.append(r[0][: done[0]])
        local = np.concatenate(recs) if recs else np.zeros(0, abi.record_dtype())
        t = torch.from_numpy(local.view(np.uint8).copy())
        got = gather_bytes(t, dist, dst=0)
        if rank == 0:
            allrec = np.concatenate([g.numpy().view(abi.record_dtype()) for g in got])
            result_q.put(allrec.tobytes())
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_equals_single_process():
    import oracle
    from paper_1907_00463_b200 import abi
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = np.frombuffer(out, abi.record_dtype())
    # single-process reference: all 6 channels in order
    fs = 2.048e6
    rng = np.random.default_rng(0)
    x = (rng.uniform(-1, 1, 2048 * 12) + 1j * rng.uniform(-1, 1, 2048 * 12))
    want = []
    for p in range(1, 7):
        ch = oracle.init_channel(p, 100.0 * p, 0, 37 * p, 0, fs)
        _, done, r, _ = oracle.track_run([ch], [0], [x], 2048, abi.TrackingCfg.default(),
                                         abi.Taps.epl(0.5), fs, 8)
        want.append(r[0][: done[0]])
    want = np.concatenate(want)
    assert got.tobytes() == want.tobytes()


def _worker_prn_split(rank, world, port, result_q):
    """Config-5 split: rank 0 synthesizes the recording and broadcasts it
    (broadcast_stream); every rank searches its PRN shard (the oracle grid
    stands in for the GPU kernel here); the planes are gathered to rank 0."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1907_00463_b200 import abi
        from paper_1907_00463_b200.shard import broadcast_stream
        fs, N = 2.046e6, 2046
        buf = torch.zeros(2 * N * 2, dtype=torch.uint8)
        if rank == 0:
            buf = torch.from_numpy(np.random.default_rng(3).integers(0, 256, 2 * N * 2, dtype=np.uint8))
        buf = broadcast_stream(buf, dist, src=0)
        x = oracle.ingest(buf.numpy(), abi.FMT_INT8_IQ, fs)
        bins = np.array([-500.0, 0.0, 500.0])
        mine = shard_list([3, 8, 17, 30, 31], world, rank)
        planes = [oracle.search_grid(x, N, 2, p, fs, bins, 1, N) for p in mine]
        local = np.stack(planes) if planes else np.zeros((0, bins.size, N))
        got = gather_bytes(torch.from_numpy(local.reshape(-1).view(np.uint8).copy()), dist, dst=0)
        if rank == 0:
            result_q.put((buf.numpy().tobytes(), np.concatenate([g.numpy() for g in got]).tobytes()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_prn_split_equals_single_process():
    import oracle
    from paper_1907_00463_b200 import abi
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_prn_split, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    stream, planes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    fs, N = 2.046e6, 2046
    raw = np.random.default_rng(3).integers(0, 256, 2 * N * 2, dtype=np.uint8)
    assert stream == raw.tobytes()  # every rank searched the broadcast bytes
    x = oracle.ingest(raw, abi.FMT_INT8_IQ, fs)
    bins = np.array([-500.0, 0.0, 500.0])
    want = np.stack([oracle.search_grid(x, N, 2, p, fs, bins, 1, N) for p in [3, 8, 17, 30, 31]])
    assert np.frombuffer(planes, np.float64).tobytes() == want.reshape(-1).tobytes()
