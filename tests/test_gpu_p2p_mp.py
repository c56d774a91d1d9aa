"""The peer-memory exchange across real processes: two
ranks on the same GPU, a gloo process group for the handle exchange only, the
exchange buffers mapped into the other process with CUDA IPC, and the phases
ordered by the device-side signals.  Each rank checks its results against the
oracle run on the union batch in (rank, index) order."""
import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist

    import gen
    import oracle
    from paper_2510_15095_b200 import u8, u32
    from paper_2510_15095_b200.sharded import P2PShardedHive
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        region = 5000
        sh = P2PShardedHive(64 * 32, region, resize_k=16)
        ref = oracle.OracleTable(64 * 32 * world, resize_k=16)
        rng = np.random.default_rng(77)                    # same stream on every rank
        for b in range(5):
            sizes = [int(x) for x in rng.integers(0, region + 1, world)]
            n = sum(sizes)
            keys = rng.integers(0, 4000 * world, n, dtype=np.uint64).astype(np.uint32)
            vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            ops = gen.bernoulli_ops(n, 0.45, 0.2, seed=b).astype(np.uint8)
            lo = sum(sizes[:rank])
            sl = slice(lo, lo + sizes[rank])
            vo, r = sh.mixed(u8(ops[sl]), u32(keys[sl]), u32(vals[sl]))
            ev, er = ref.mixed(ops, keys, vals)
            assert (r.cpu().numpy() == er[sl]).all(), f"batch {b}: results"
            assert (vo.cpu().numpy().astype(np.uint32) == ev[sl]).all(), f"batch {b}: values"
        torch.cuda.synchronize()
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
        out.put((rank, "ok"))
    except Exception as e:                                  # report, do not hang the parent
        out.put((rank, repr(e)))


def test_p2p_exchange_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert res == {0: "ok", 1: "ok"}, res
