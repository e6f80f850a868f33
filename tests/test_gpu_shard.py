"""Device path of the multi-GPU split (paper_2509_07120_b200/shard.py) on one
B200.

The box has one GPU, so:
* ranks are emulated by running each rank's device steps in turn on cuda:0
  and combining them the way the collectives would;
* a real world-size-1 process group runs the public entry point end to end.
The bar is bit-identity with the single-GPU call: every row is computed by
the same kernel, in the same key order.
"""

import os
import socket

import numpy as np
import pytest

from golden_inputs import make_qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _setup(bsa, frames=5, patches=600, heads=2, tau=0.4, rho=0.8, seed=5):
    import torch
    lay = bsa.TokenLayout(frames, patches, 5)
    q, k, v = (torch.from_numpy(x).to("cuda", torch.bfloat16)
               for x in make_qkv(heads, lay.total_tokens, 64, seed))
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    return lay, q, k, v, bsa.MaskPolicy(tau, rho, g)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_emulated_ranks_bit_identical(bsa, world):
    import torch
    from paper_2509_07120_b200.shard import DeviceOps, ShardPlan

    lay, q, k, v, pol = _setup(bsa)
    g = pol.geometry
    ref_mask = bsa.predict_mask(q, k, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, ref_mask))

    ops = DeviceOps()
    plan = ShardPlan(lay, world)
    qp, kp = ops.pool(q, lay, 128), ops.pool(k, lay, 64)
    bits, counts = [], []
    for r in range(world):
        qb0, qb1 = plan.qblock_range(r)
        b, c = ops.score_rows(qp[:, qb0:qb1], kp, 64, pol)
        bits.append(b)
        counts.append(c)
    bits = torch.cat(bits, dim=1).reshape(-1, bits[0].shape[2])
    counts = torch.cat(counts, dim=1).reshape(-1)
    assert torch.equal(bits, ref_mask.device_bits()), "row-split scoring changed the mask"
    assert torch.equal(counts, ref_mask.device_counts())

    mask = bsa.BlockMask._from_device(bits, counts, q.shape[0], g)
    acc = torch.zeros_like(ref)
    for r in range(world):
        acc += ops.attend(q, k, v, lay, mask, r, world)  # the all-reduce(sum)
    assert torch.equal(acc, ref)
    for r in range(world):
        t0, t1 = plan.token_range(r)
        assert torch.equal(acc[:, t0:t1], ref[:, t0:t1])


def test_schedule_is_deterministic(bsa):
    """Every rank builds the LPT list independently: shards must agree."""
    import torch
    lay, q, k, v, pol = _setup(bsa, frames=3, patches=1369, heads=3, tau=0.9, rho=0.5)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    job = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
    first = [bsa.sparse_attention(job, shard=s, num_shards=4) for s in range(4)]
    for _ in range(3):
        for s in range(4):
            assert torch.equal(bsa.sparse_attention(job, shard=s, num_shards=4), first[s])


def test_world1_process_group_end_to_end(bsa):
    import torch
    import torch.distributed as dist
    from paper_2509_07120_b200.shard import sharded_sparse_attention

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay, q, k, v, pol = _setup(bsa)
        out, mask = sharded_sparse_attention(q, k, v, lay, pol, return_mask=True)
        ref_mask = bsa.predict_mask(q, k, pol, layout=lay)
        ref = bsa.sparse_attention(
            bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, ref_mask))
        assert torch.equal(mask.device_bits(), ref_mask.device_bits())
        assert torch.equal(out, ref)
        out2, mask2 = sharded_sparse_attention(q, k, v, lay, pol, return_mask=True,
                                               chunk_heads=1)  # per-head pipeline
        assert torch.equal(out2, ref)
        assert torch.equal(mask2.device_bits(), ref_mask.device_bits())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 3])
def test_scatter_epilogue_emulated_ranks(bsa, world):
    """The fused combine: the kernel epilogue stores each row into the buffer
    of the rank owning its frame (here: `world` buffers on one GPU, reached
    through the same pointer table the NVLink peers use)."""
    import torch
    from paper_2509_07120_b200.shard import DeviceOps, ShardPlan

    lay, q, k, v, pol = _setup(bsa, frames=6, heads=3)
    ref_mask = bsa.predict_mask(q, k, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, ref_mask))
    plan = ShardPlan(lay, world)
    H, T, d = q.shape
    bufs = [torch.full((H, plan.token_range(r)[1] - plan.token_range(r)[0], d), float("nan"),
                       dtype=torch.bfloat16, device="cuda") for r in range(world)]

    class Target:  # what ScatterTarget provides, minus the IPC
        pass
    t = Target()
    t.world = world
    t.token_begin = torch.tensor([plan.token_range(r)[0] for r in range(world)] + [T],
                                 dtype=torch.int64, device="cuda")
    t.chunk_ptrs = lambda head0: torch.tensor(
        [b.data_ptr() + head0 * b.shape[1] * d * 2 for b in bufs], dtype=torch.int64,
        device="cuda")
    ops = DeviceOps()
    # every shard of a 2-way LPT split, and a per-head chunked call
    for s in range(2):
        ops.attend_scatter(q, k, v, lay, ref_mask, s, 2, t)
    torch.cuda.synchronize()
    for r in range(world):
        t0, t1 = plan.token_range(r)
        assert torch.equal(bufs[r], ref[:, t0:t1]), f"rank {r} buffer differs"
    for b in bufs:
        b.fill_(float("nan"))
    for h in range(H):
        m_h = bsa.BlockMask._from_device(ref_mask.device_bits()[h * ref_mask.geometry.nq_blocks:
                                                               (h + 1) * ref_mask.geometry.nq_blocks],
                                         ref_mask.device_counts()[h * ref_mask.geometry.nq_blocks:
                                                                  (h + 1) * ref_mask.geometry.nq_blocks],
                                         1, ref_mask.geometry)
        ops.attend_scatter(q[h:h + 1], k[h:h + 1], v[h:h + 1], lay, m_h, 0, 1, t, head0=h)
    torch.cuda.synchronize()
    for r in range(world):
        t0, t1 = plan.token_range(r)
        assert torch.equal(bufs[r], ref[:, t0:t1])


def test_world1_scatter_combine(bsa):
    import torch
    import torch.distributed as dist
    from paper_2509_07120_b200.shard import ScatterTarget, ShardPlan, sharded_sparse_attention

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay, q, k, v, pol = _setup(bsa)
        ref_mask = bsa.predict_mask(q, k, pol, layout=lay)
        ref = bsa.sparse_attention(
            bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, ref_mask))
        out = sharded_sparse_attention(q, k, v, lay, pol, combine="scatter")
        assert torch.equal(out, ref)
        tgt = ScatterTarget(ShardPlan(lay, 1), q.shape[0], q.shape[2], 0)
        for _ in range(2):  # persistent target reused across layers, chunked
            out2 = sharded_sparse_attention(q, k, v, lay, pol, combine="scatter",
                                            scatter_target=tgt, chunk_heads=1)
            assert torch.equal(out2, ref)
        tgt.close()
        with pytest.raises(ValueError):
            sharded_sparse_attention(q, k, v, lay, pol, combine="scatter", inputs="replicated")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("combine", ["allreduce", "scatter"])
def test_emulated_8_ranks_config5(bsa, combine):
    """BASELINE config 5's split at its size: N=1000 frames, rho=0.75, 2 heads,
    8 emulated ranks on one GPU. Each rank scores its q-block rows and
    attends its share of every head's LPT rows (the automatic key-range
    split engages at this size); the combined output and the gathered mask
    must be bit-identical to the single-GPU call."""
    import torch
    from paper_2509_07120_b200.shard import DeviceOps, ShardPlan

    world = 8
    lay = bsa.TokenLayout(1000, 1369, 5)
    H, T, d = 2, lay.total_tokens, 64
    gen = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn((H, T, d), generator=gen, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
    ref_mask = bsa.predict_mask(q, k, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, ref_mask))

    ops = DeviceOps()
    plan = ShardPlan(lay, world)
    qp, kp = ops.pool(q, lay, 128), ops.pool(k, lay, 64)
    bits, counts = [], []
    for r in range(world):
        qb0, qb1 = plan.qblock_range(r)
        b, c = ops.score_rows(qp[:, qb0:qb1], kp, d, pol)
        bits.append(b)
        counts.append(c)
    bits = torch.cat(bits, dim=1).reshape(-1, bits[0].shape[2])
    counts = torch.cat(counts, dim=1).reshape(-1)
    assert torch.equal(bits, ref_mask.device_bits()), "row-split scoring changed the mask"
    assert torch.equal(counts, ref_mask.device_counts())
    mask = bsa.BlockMask._from_device(bits, counts, H, pol.geometry)

    if combine == "allreduce":
        acc = torch.zeros_like(ref)
        for r in range(world):
            acc += ops.attend(q, k, v, lay, mask, r, world)  # the sum all-reduce
        assert torch.equal(acc, ref)
    else:
        bufs = [torch.full((H, plan.token_range(r)[1] - plan.token_range(r)[0], d), float("nan"),
                           dtype=torch.bfloat16, device="cuda") for r in range(world)]

        class Target:  # ScatterTarget's pointer table, minus the IPC
            pass
        t = Target()
        t.world = world
        t.token_begin = torch.tensor([plan.token_range(r)[0] for r in range(world)] + [T],
                                     dtype=torch.int64, device="cuda")
        t.chunk_ptrs = lambda head0: torch.tensor(
            [b.data_ptr() + head0 * b.shape[1] * d * 2 for b in bufs], dtype=torch.int64,
            device="cuda")
        for r in range(world):
            ops.attend_scatter(q, k, v, lay, mask, r, world, t)
        torch.cuda.synchronize()
        for r in range(world):
            t0, t1 = plan.token_range(r)
            assert torch.equal(bufs[r], ref[:, t0:t1]), f"rank {r} rows differ"
