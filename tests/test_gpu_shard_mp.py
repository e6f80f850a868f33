"""The multi-GPU path with REAL separate processes, on the one GPU of the test
box: two ranks over gloo (NCCL refuses two ranks on one device), both on
cuda:0. This exercises what the single-process tests cannot:
* the frame-sharded all-gathers of CUDA tensors between processes;
* row-split scoring with the mask all-gather;
* the fused output scatter through CUDA IPC: each rank maps the other's
  output buffer (bsa_ipc_open across processes) and the attention epilogue
  stores rows into it.
Each rank's result must equal the single-process device result bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, combine, chunk, q_out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2509_07120_b200 as bsa
        from golden_inputs import make_qkv
        from paper_2509_07120_b200.shard import ShardPlan, sharded_sparse_attention

        lay = bsa.TokenLayout(5, 600, 5)
        q, k, v = (torch.from_numpy(x).to("cuda", torch.bfloat16)
                   for x in make_qkv(2, lay.total_tokens, 64, 9))
        pol = bsa.MaskPolicy(0.4, 0.8, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
        t0, t1 = ShardPlan(lay, world).token_range(rank)
        out = sharded_sparse_attention(q[:, t0:t1].contiguous(), k[:, t0:t1].contiguous(),
                                       v[:, t0:t1].contiguous(), lay, pol, combine=combine,
                                       chunk_heads=chunk)
        mask = bsa.predict_mask(q, k, pol, layout=lay)
        ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
        q_out.put((rank, bool(torch.equal(out, ref[:, t0:t1])), None))
    except Exception as e:  # report instead of hanging the parent
        q_out.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("combine,chunk", [("allreduce", None), ("scatter", None),
                                           ("scatter", 1), ("reduce_scatter", 2)])
def test_two_process_ranks_on_one_gpu(combine, chunk):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = here + os.pathsep + os.environ.get("PYTHONPATH", "")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, combine, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, ok, err = q.get(timeout=300)
        res[r] = (ok, err)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert res[r][0], f"rank {r}: {res[r][1]}"


def _stack_worker(rank, world, port, combine, q_out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2509_07120_b200 as bsa
        from paper_2509_07120_b200.shard import ShardPlan
        from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for

        lay = bsa.TokenLayout(4, 700, 5)
        stack = GlobalAttentionStack(layers=2, seed=4)
        g = torch.Generator(device="cuda").manual_seed(6)
        x = torch.randn((lay.total_tokens, stack.dim), generator=g, device="cuda").to(torch.bfloat16)
        pol = policy_for(lay, 0.0, 0.75)
        t0, t1 = ShardPlan(lay, world).token_range(rank)
        y = stack.forward_sharded(x[t0:t1].contiguous(), lay, pol, combine=combine)
        ref = stack(x, lay, pol, "sparse")
        q_out.put((rank, bool(torch.equal(y, ref[t0:t1])), None))
    except Exception as e:  # report instead of hanging the parent
        q_out.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("combine", ["scatter", "reduce_scatter"])
def test_two_process_stack_on_one_gpu(combine):
    """Config 3 with the frames split over two real processes: each rank's
    rows of a 2-layer stack equal the single-process stack bit for bit."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = here + os.pathsep + os.environ.get("PYTHONPATH", "")
    procs = [ctx.Process(target=_stack_worker, args=(r, 2, port, combine, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, ok, err = q.get(timeout=300)
        res[r] = (ok, err)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert res[r][0], f"rank {r}: {res[r][1]}"
