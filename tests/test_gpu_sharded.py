"""The sharded path on one GPU: route kernel -> NCCL all-to-all (world size 1)
-> local phases -> inverse all-to-all -> unroute, against a plain table."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import gen

pytestmark = pytest.mark.gpu


def test_sharded_world1_nccl_matches_plain_table():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2510_15095_b200 import HiveTable, u8, u32
    from paper_2510_15095_b200.sharded import ShardedHive
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = ShardedHive(256 * 32, resize_k=16)
        ref = HiveTable(256 * 32, resize_k=16)
        rng = np.random.default_rng(9)
        for b in range(5):
            n = 20000
            keys = u32(rng.integers(0, 30000, n, dtype=np.uint64).astype(np.uint32))
            vals = u32(rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32))
            ops = u8(gen.bernoulli_ops(n, 0.5, 0.2, seed=b))
            vo1, r1 = sh.mixed(ops, keys, vals)
            vo2, r2 = ref.mixed(ops, keys, vals)
            assert torch.equal(r1.cpu(), r2.cpu()) and torch.equal(vo1.cpu(), vo2.cpu())
        q = u32(rng.integers(0, 40000, 50000, dtype=np.uint64).astype(np.uint32))
        v1, f1 = sh.find(q)
        v2, f2 = ref.find(q)
        assert torch.equal(f1.cpu(), f2.cpu()) and torch.equal(v1.cpu(), v2.cpu())
        e1 = sh.erase(q[:1000])
        e2 = ref.erase(q[:1000])
        assert torch.equal(e1.cpu(), e2.cpu())
        st1 = sh.insert(q[:5000], q[:5000])
        st2 = ref.insert(q[:5000], q[:5000])
        assert torch.equal(st1.cpu(), st2.cpu())
    finally:
        dist.destroy_process_group()
