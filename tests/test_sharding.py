"""N-sharded linear on 2 ranks over gloo (CPU): the channel split, the
all-gather reassembly (M=1 and M>1, equal and unequal shards) and bit-identity
with the unsharded result.  The per-rank compute of the CPU test is the oracle standing in
for the GPU engine; the -m gpu test runs the same sharding over the engine itself
(two ranks sharing the one GPU of a gpurun box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import COracle
    from paper_2408_08554_b200.sharded import ShardedLinear, shard_bounds
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    orc = COracle()
    try:
        for (m, n, k, wbits, abits, seed) in cases:
            rng = np.random.default_rng(seed)
            x = rng.standard_normal((m, k)).astype(np.float16).astype(np.float64)
            wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
            sb = rng.uniform(1e-3, 1e-2, n)
            zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
            lo, hi = shard_bounds(n, world)[rank]
            ac, sa, za = orc.quantize(x, abits, 0, 2)

            def local(xx, lo=lo, hi=hi, ac=ac, sa=sa, za=za, wc=wc, sb=sb, zb=zb):
                y = orc.quantized_linear(ac, abits, sa, za, wc[lo:hi], wbits, sb[lo:hi], zb[lo:hi])
                return torch.from_numpy(y)

            lin = ShardedLinear(local_fn=local, n_full=n)
            y = lin(None).numpy()
            full = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb)
            q.put((rank, m, n, bool(np.array_equal(y, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_linear_gloo(world):
    cases = [(1, 128, 256, 2, 8, 1), (4, 100, 320, 4, 4, 2), (3, 77, 64, 3, 5, 3), (1, 64, 128, 8, 8, 4)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world * len(cases))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for (_, _, _, ok) in results), results


def test_shard_bounds_cover_channels():
    from paper_2408_08554_b200.sharded import shard_bounds
    for n in (1, 7, 640, 1728, 11008, 28672):
        for g in (1, 2, 4, 8):
            b = shard_bounds(n, g)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(g - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1


def _engine_worker(rank, world, port, q):
    """two ranks on one GPU, gloo collective: ShardedLinear over the ENGINE
    (PackedWeights.shard + Linear on each rank's channel slice) vs the
    unsharded engine Linear, bit for bit."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2408_08554_b200 as abq
    from paper_2408_08554_b200.sharded import ShardedLinear
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        for (m, n, k, wbits, abits, seed) in [(1, 1728, 5120, 2, 8, 1), (4, 1000, 2048, 4, 4, 2),
                                              (64, 1024, 8192, 4, 4, 3)]:
            rng = np.random.default_rng(seed)
            wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
            sb = rng.uniform(1e-3, 1e-2, n)
            zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
            x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
            w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
            spec = abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN)
            y = ShardedLinear(w, spec, max_m=m)(x, out_dtype=torch.float64)
            full = abq.Linear(w, spec, max_m=m)(x, out_dtype=torch.float64)
            q.put((rank, m, n, bool(torch.equal(y.cpu(), full.cpu()))))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_engine_linear_gloo_two_ranks_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2 * 3)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for (*_, ok) in results), results
