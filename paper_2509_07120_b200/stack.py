"""Model harness for BASELINE.json config 3: a stack of VGGT-aggregator
global-attention blocks with random-init weights, each block's dense global
attention replaced by the block-sparse operator (arXiv 2509.07120 retrofit).

The reference package has no model code. This harness builds the
smallest faithful block around the path: pre-LayerNorm, fused QKV
projection, per-head attention over the whole multi-frame token sequence, an
output projection and a residual. It also has an optional MLP. The GEMMs are
plain cuBLAS (torch.nn.functional.linear); the attention is
``predict_mask`` + ``sparse_attention`` from this package
(``mode="sparse"``), or cuDNN SDPA (``mode="dense"``) as the baseline.

Tokens are (T, C) in the interleaved VGGT order (per frame: S special tokens,
then P patches, layout.py:27-66). C = heads x head_dim = 16 x 64 = 1024.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .dense import AttentionInputs
from .layout import BlockGeometry, TokenLayout, partition_permutation
from .maskpred import MaskPolicy, predict_mask, predict_mask_pooled
from .qkv import proj_residual, qkv_projection
from .sparse import SparseAttentionJob, sparse_attention


@dataclass
class BlockWeights:
    ln_w: torch.Tensor
    ln_b: torch.Tensor
    qkv_w: torch.Tensor  # (3C, C)
    qkv_b: torch.Tensor
    proj_w: torch.Tensor  # (C, C)
    proj_b: torch.Tensor
    mlp: tuple | None = None  # (ln_w, ln_b, fc1_w, fc1_b, fc2_w, fc2_b)


class GlobalAttentionStack:
    """`layers` global-attention blocks of width heads*head_dim, random init
    (seeded): weights ~ N(0, 1/C), biases 0, LayerNorm identity."""

    def __init__(self, layers: int = 24, heads: int = 16, head_dim: int = 64, mlp: bool = False,
                 seed: int = 0, device="cuda", dtype=torch.bfloat16):
        self.heads, self.head_dim = heads, head_dim
        C = heads * head_dim
        self.dim = C
        g = torch.Generator(device="cpu").manual_seed(seed)

        def w(o, i):
            return (torch.randn((o, i), generator=g) / math.sqrt(i)).to(device, dtype)

        self.blocks = []
        for _ in range(layers):
            mlp_w = None
            if mlp:
                mlp_w = (torch.ones(C, device=device, dtype=dtype), torch.zeros(C, device=device, dtype=dtype),
                         w(4 * C, C), torch.zeros(4 * C, device=device, dtype=dtype),
                         w(C, 4 * C), torch.zeros(C, device=device, dtype=dtype))
            self.blocks.append(BlockWeights(
                torch.ones(C, device=device, dtype=dtype), torch.zeros(C, device=device, dtype=dtype),
                w(3 * C, C), torch.zeros(3 * C, device=device, dtype=dtype),
                w(C, C), torch.zeros(C, device=device, dtype=dtype), mlp_w))

    def attention(self, x: torch.Tensor, blk: BlockWeights, layout: TokenLayout,
                  policy: MaskPolicy | None, mode: str) -> torch.Tensor:
        T, C = x.shape
        H, d = self.heads, self.head_dim
        h = F.layer_norm(x, (C,), blk.ln_w, blk.ln_b)
        qkv = F.linear(h, blk.qkv_w, blk.qkv_b)                       # (T, 3C)
        qkv = qkv.view(T, 3, H, d).permute(1, 2, 0, 3)                # (3, H, T, d) view
        q, k, v = qkv[0], qkv[1], qkv[2]                              # token stride 3C
        if mode == "sparse":
            mask = predict_mask(q, k, policy, layout=layout)
            o = sparse_attention(SparseAttentionJob(AttentionInputs(q, k, v), layout, mask))
        elif mode == "dense":
            o = F.scaled_dot_product_attention(q[None], k[None], v[None])[0]
        else:
            raise ValueError(f"mode must be 'sparse' or 'dense', got {mode!r}")
        o = o.permute(1, 0, 2).reshape(T, C)
        return F.linear(o, blk.proj_w, blk.proj_b)

    def forward(self, x: torch.Tensor, layout: TokenLayout, policy: MaskPolicy | None = None,
                mode: str = "sparse") -> torch.Tensor:
        if x.shape != (layout.total_tokens, self.dim):
            raise ValueError(f"x must be ({layout.total_tokens}, {self.dim}), got {tuple(x.shape)}")
        if mode in ("sparse", "fused") and policy is None:
            raise ValueError(f"{mode} mode needs a MaskPolicy")
        if mode == "fused":
            return self._forward_fused(x, layout, policy)
        for blk in self.blocks:
            x = x + self.attention(x, blk, layout, policy, mode)
            if blk.mlp is not None:
                lw, lb, w1, b1, w2, b2 = blk.mlp
                h = F.layer_norm(x, (self.dim,), lw, lb)
                x = x + F.linear(F.gelu(F.linear(h, w1, b1)), w2, b2)
        return x

    __call__ = forward

    def attention_fused(self, xp: torch.Tensor, blk: BlockWeights, layout: TokenLayout,
                        policy: MaskPolicy) -> torch.Tensor:
        """One block's attention branch with tokens in partitioned order
        [specials | patches]: LayerNorm, then the tensor-core QKV projection
        whose epilogue writes head-major Q/K/V plus the pooled patch Q/K
        (qkv.qkv_projection), predict_mask_pooled (no pooling pass), the
        block-sparse kernel on the in-place permuted inputs (no pack pass),
        and the output projection (cuBLAS here; the fused stack uses
        qkv.proj_residual, which also adds the residual).  Same mask as mode="sparse" on the same
        Q/K; Q/K/V themselves come from this GEMM instead of cuBLAS."""
        T, C = xp.shape
        o = self._attend_fused(xp, blk, layout, policy)
        return F.linear(o.permute(1, 0, 2).reshape(T, C), blk.proj_w, blk.proj_b)

    def _attend_fused(self, xp, blk, layout, policy):
        """LayerNorm -> fused QKV projection (+ pooled Q/K) -> scoring from
        the pools -> block-sparse attention on the head-major partitioned
        Q/K/V; returns the (H, T, 64) output, partitioned order."""
        C = xp.shape[1]
        h = F.layer_norm(xp, (C,), blk.ln_w, blk.ln_b)
        q, k, v, qp, kp = qkv_projection(h, blk.qkv_w, blk.qkv_b, self.heads, layout,
                                         policy.geometry)
        mask = predict_mask_pooled(qp, kp, policy, validate=False)
        return sparse_attention(SparseAttentionJob(AttentionInputs(q, k, v, validate=False), layout,
                                                   mask), inputs_permuted=True)

    def _forward_fused(self, x: torch.Tensor, layout: TokenLayout, policy: MaskPolicy):
        # every op but attention acts per token: keep the residual stream in
        # partitioned order for the whole stack, permute once each way
        perm, inv = partition_permutation(layout)
        perm_t = torch.from_numpy(perm).to(x.device)
        inv_t = torch.from_numpy(inv).to(x.device)
        xp = x.index_select(0, perm_t)
        for blk in self.blocks:
            # output projection + bias + residual in one GEMM reading the
            # head-major attention output in place (qkv.proj_residual)
            o = self._attend_fused(xp, blk, layout, policy)
            xp = proj_residual(o, blk.proj_w, blk.proj_b, xp)
            if blk.mlp is not None:
                lw, lb, w1, b1, w2, b2 = blk.mlp
                h = F.layer_norm(xp, (self.dim,), lw, lb)
                xp = xp + F.linear(F.gelu(F.linear(h, w1, b1)), w2, b2)
        return xp.index_select(0, inv_t)

    def forward_sharded(self, x_local: torch.Tensor, layout: TokenLayout, policy: MaskPolicy, *,
                        group=None, comm_group=None, combine: str = "auto",
                        chunk_heads: int | None = None, ops=None) -> torch.Tensor:
        """The stack with the frames split over the ranks of `group` (config 3
        at 2/4/8 GPUs): each rank holds the tokens of its frames
        (ShardPlan.token_range), shape (T_r, C).  LayerNorm, the QKV / output
        projections, the residual and the MLP act per token and run locally;
        the global attention is shard.sharded_sparse_attention (NCCL
        all-gather of Q/K/V, row-split scoring, every rank attends its share
        of each head's rows, rows returned to their owners).  With the
        scatter combine one ScatterTarget (CUDA IPC mapping) serves every
        layer.  Returns this rank's (T_r, C) output; with one rank it equals
        forward() bit for bit."""
        from .shard import ScatterTarget, ShardPlan, _rank_world, sharded_sparse_attention

        rank, world = _rank_world(group)
        plan = ShardPlan(layout, world, policy.geometry.block_q, policy.geometry.block_k)
        t0, t1 = plan.token_range(rank)
        if x_local.shape != (t1 - t0, self.dim):
            raise ValueError(f"rank {rank} must hold ({t1 - t0}, {self.dim}) tokens, "
                             f"got {tuple(x_local.shape)}")
        H, d, C = self.heads, self.head_dim, self.dim
        Tr = t1 - t0
        target = None
        if combine in ("auto", "scatter") and ops is None and x_local.device.type == "cuda":
            combine = "scatter"
            target = ScatterTarget(plan, H, d, rank, group, x_local.device)
        x = x_local
        try:
            for blk in self.blocks:
                h = F.layer_norm(x, (C,), blk.ln_w, blk.ln_b)
                qkv = F.linear(h, blk.qkv_w, blk.qkv_b).view(Tr, 3, H, d).permute(1, 2, 0, 3)
                o = sharded_sparse_attention(qkv[0], qkv[1], qkv[2], layout, policy, group=group,
                                             inputs="sharded", ops=ops, chunk_heads=chunk_heads,
                                             comm_group=comm_group, combine=combine,
                                             scatter_target=target)
                o = o.permute(1, 0, 2).reshape(Tr, C)
                x = x + F.linear(o, blk.proj_w, blk.proj_b)
                if blk.mlp is not None:
                    lw, lb, w1, b1, w2, b2 = blk.mlp
                    hm = F.layer_norm(x, (C,), lw, lb)
                    x = x + F.linear(F.gelu(F.linear(hm, w1, b1)), w2, b2)
        finally:
            if target is not None:
                torch.cuda.current_stream(x_local.device).synchronize()
                target.close(group)
        return x

    def layer_statistics(self, x: torch.Tensor, layout: TokenLayout,
                         policy: MaskPolicy | None = None, mode: str = "sparse") -> list[dict]:
        """The paper's per-layer attention analysis (§4.x "Visualizing
        Attention Maps": mean / max attention of the special/patch quadrants
        against layer index), streamed on the GPU without any T x T map
        (analysis.py). With a policy, each layer also reports the mean
        fraction of patch attention mass its predicted mask keeps
        (mask_recall), the per-layer tau/rho selection signal. The stack runs
        forward in `mode` while the statistics are taken."""
        from .analysis import attention_quadrant_stats, block_attention_map, mask_recall

        if x.shape != (layout.total_tokens, self.dim):
            raise ValueError(f"x must be ({layout.total_tokens}, {self.dim}), got {tuple(x.shape)}")
        T, C = x.shape
        H, d = self.heads, self.head_dim
        rows = []
        for i, blk in enumerate(self.blocks):
            h = F.layer_norm(x, (C,), blk.ln_w, blk.ln_b)
            qkv = F.linear(h, blk.qkv_w, blk.qkv_b).view(T, 3, H, d).permute(1, 2, 0, 3)
            inp = AttentionInputs(qkv[0], qkv[1], qkv[2])
            st = attention_quadrant_stats(inp, layout)
            row = {"layer": i, "means": st.means, "maxes": st.maxes}
            if policy is not None:
                mask = predict_mask(qkv[0], qkv[1], policy, layout=layout)
                row["recall"] = float(mask_recall(block_attention_map(inp, layout), mask).mean())
            rows.append(row)
            x = x + self.attention(x, blk, layout, policy, mode)
            if blk.mlp is not None:
                lw, lb, w1, b1, w2, b2 = blk.mlp
                hm = F.layer_norm(x, (self.dim,), lw, lb)
                x = x + F.linear(F.gelu(F.linear(hm, w1, b1)), w2, b2)
        return rows


def policy_for(layout: TokenLayout, tau: float, rho: float, block_q: int = 128,
               block_k: int = 64) -> MaskPolicy:
    return MaskPolicy(tau, rho, BlockGeometry(layout.patch_tokens, block_q, block_k))
