"""Multi-rank host logic of the frame-sharded path (paper_2509_07120_b200/
shard.py), world size 2 over gloo on CPU.

The device kernels need a B200, so these tests inject a checker-backed
``ops`` object (oracle restatement: C scoring, float64 attention). That is
test infrastructure; the product path uses DeviceOps (libbsa.so). What is
under test here is everything around the compute:
* frame ownership;
* the padded all-gathers that rebuild the sequence;
* the scoring-row split and the mask all-gather;
* the shard-disjoint output;
* the exact sum-combine;
* each rank's output slice.
The result must equal the single-process oracle bit for bit (mask) and to
float64 round-off (attention).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2509_07120_b200.layout import BlockGeometry, TokenLayout
from paper_2509_07120_b200.shard import ShardPlan

F, P, S, H, D = 5, 300, 5, 2, 64
BQ, BK = 128, 64
TAU, RHO = 0.4, 0.8


def _inputs():
    lay = TokenLayout(F, P, S)
    rng = np.random.default_rng(3)
    return lay, [rng.standard_normal((H, lay.total_tokens, D)).astype(np.float32)
                 for _ in range(3)]


class OracleOps:
    """CPU checker standing in for DeviceOps (tests only)."""

    def pool(self, x, layout, block):
        pidx = oracle.patch_indices(layout.frames, layout.patches_per_frame,
                                    layout.specials_per_frame)
        return torch.from_numpy(oracle.block_pool(x.numpy()[:, pidx], block))

    def score_rows(self, qp_rows, kp, head_dim, policy):
        h, nr, _ = qp_rows.shape
        nk = kp.shape[1]
        if nr == 0:
            return (torch.zeros((h, 0, -(-nk // 8)), dtype=torch.uint8),
                    torch.zeros((h, 0), dtype=torch.int32))
        probs = oracle.pooled_scores(qp_rows.numpy(), kp.numpy(), head_dim)
        mask, counts = oracle.select_blocks(probs, policy.tau, policy.min_blocks)
        bits = oracle.pack_bits(mask).reshape(h, nr, -1)
        return torch.from_numpy(bits), torch.from_numpy(counts)

    def attend(self, q, k, v, layout, mask, shard, num_shards):
        # shard ownership: every num_shards-th (head, token) row, any rule works
        # as long as the shards are disjoint and cover everything
        blocks = mask.blocks
        T = layout.total_tokens
        out = np.zeros((q.shape[0], T, D), dtype=np.float64)
        rows = [t for t in range(T) if t % num_shards == shard]
        res = oracle.masked_attention_f64(q.numpy(), k.numpy(), v.numpy(), layout.frames,
                                          layout.patches_per_frame, layout.specials_per_frame,
                                          blocks, BQ, BK, rows=rows)
        out[:, rows] = res
        return torch.from_numpy(out)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, inputs, result_q, chunk=None, combine="auto"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_07120_b200.maskpred import MaskPolicy
        from paper_2509_07120_b200.shard import sharded_sparse_attention

        lay, (q, k, v) = _inputs()
        pol = MaskPolicy(TAU, RHO, BlockGeometry(lay.patch_tokens, BQ, BK))
        plan = ShardPlan(lay, world, BQ, BK)
        if inputs == "sharded":
            t0, t1 = plan.token_range(rank)
            xs = [torch.from_numpy(np.ascontiguousarray(x[:, t0:t1])) for x in (q, k, v)]
        else:
            xs = [torch.from_numpy(x) for x in (q, k, v)]
        out, mask = sharded_sparse_attention(*xs, lay, pol, inputs=inputs, ops=OracleOps(),
                                             return_mask=True, chunk_heads=chunk,
                                             combine=combine)
        result_q.put((rank, out.numpy(), mask.blocks.copy()))
    finally:
        dist.destroy_process_group()


def _run(world, inputs, chunk=None, combine="auto"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, inputs, q, chunk, combine))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, blocks = q.get(timeout=240)
        res[r] = (out, blocks)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.fixture(scope="module")
def single_process():
    lay, (q, k, v) = _inputs()
    pidx = oracle.patch_indices(F, P, S)
    mask, _ = oracle.predict_mask(q[:, pidx], k[:, pidx], BQ, BK, TAU, RHO)
    ref = oracle.masked_attention_f64(q, k, v, F, P, S, mask, BQ, BK)
    return lay, mask, ref


@pytest.mark.parametrize("world", [2, 3])
def test_frame_sharded_matches_single_process(world, single_process):
    lay, mask, ref = single_process
    res = _run(world, "sharded")
    plan = ShardPlan(lay, world, BQ, BK)
    for r, (out, blocks) in res.items():
        assert np.array_equal(blocks, mask), f"rank {r}: gathered mask differs"
        t0, t1 = plan.token_range(r)
        assert out.shape == (H, t1 - t0, D)
        np.testing.assert_allclose(out, ref[:, t0:t1], rtol=0, atol=1e-12)


def test_head_chunked_pipeline_matches(single_process):
    """chunk_heads=1: per-head async gathers / all-reduces, same result."""
    lay, mask, ref = single_process
    res = _run(2, "sharded", chunk=1)
    plan = ShardPlan(lay, 2, BQ, BK)
    for r, (out, blocks) in res.items():
        assert np.array_equal(blocks, mask)
        t0, t1 = plan.token_range(r)
        np.testing.assert_allclose(out, ref[:, t0:t1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("world,chunk", [(2, None), (3, 1)])
def test_reduce_scatter_combine(world, chunk, single_process):
    """combine="reduce_scatter": rows staged by owner, one NCCL-style
    reduce-scatter (sum of disjoint rows) per head chunk."""
    lay, mask, ref = single_process
    res = _run(world, "sharded", chunk=chunk, combine="reduce_scatter")
    plan = ShardPlan(lay, world, BQ, BK)
    for r, (out, blocks) in res.items():
        assert np.array_equal(blocks, mask)
        t0, t1 = plan.token_range(r)
        assert out.shape == (H, t1 - t0, D)
        np.testing.assert_allclose(out, ref[:, t0:t1], rtol=0, atol=1e-12)


def test_replicated_inputs_return_full_output(single_process):
    lay, mask, ref = single_process
    res = _run(2, "replicated")
    for r, (out, blocks) in res.items():
        assert np.array_equal(blocks, mask)
        np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)


def test_shard_plan_ownership():
    lay = TokenLayout(7, 1369, 5)
    plan = ShardPlan(lay, 3)
    frames = [plan.frame_range(r) for r in range(3)]
    assert frames == [(0, 3), (3, 5), (5, 7)]
    toks = [plan.token_range(r) for r in range(3)]
    assert toks[0][0] == 0 and toks[-1][1] == lay.total_tokens
    assert all(toks[i][1] == toks[i + 1][0] for i in range(2))
    g = plan.geometry
    rows = [plan.qblock_range(r) for r in range(3)]
    assert rows[0][0] == 0 and rows[-1][1] == g.nq_blocks
    assert all(rows[i][1] == rows[i + 1][0] for i in range(2))
    with pytest.raises(ValueError):
        ShardPlan(TokenLayout(2, 10, 1), 3)
    with pytest.raises(ValueError):
        ShardPlan(lay, 0)
