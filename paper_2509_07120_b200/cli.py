"""Command-line interface, B200 edition of the reference's ``bsattn`` CLI
(/root/reference/pkg/src/bsattn/cli.py:237-330).

The hot-path subcommands keep the reference's flags, files and CSV output,
so its flows (tests/test_cli.py:44-112) run unchanged on the GPU:

    mask    .bsat q/k -> .bsm block mask (+ --stats per-head sparsity CSV)
    attend  .bsat q/k/v (+ .bsm) -> .bsat output, dense or block-sparse
            (+ --report per-head CSV)
    bench   dense vs sparse sweep, reference CSV schema (+ --with-predict)
    analyze quadrant statistics, reference CSV schema: of a materialised
            --map (as the reference), or streamed from --q/--k without the
            map (analysis.py)

``correspond``, ``layerdrop`` and ``synth`` work on materialised attention
maps or generate inputs. They are outside the data-parallel path (SURVEY.md
§2.1) and exit with a message.
"""

from __future__ import annotations

import argparse
import csv
import sys

from .benchsweep import bench_sweep, write_bench_csv
from .dense import AttentionInputs, dense_attention
from .layout import BlockGeometry, TokenLayout, patch_token_indices
from .maskpred import MaskPolicy, predict_mask, read_mask, write_mask
from .sparse import SparseAttentionJob, sparse_attention, sparse_attention_stats
from .tensorio import read_tensor, write_tensor

OUT_OF_SCOPE = ("correspond", "layerdrop", "synth")


def _fmt(x: float) -> str:
    return f"{x:.6g}"


def _layout_flags(p: argparse.ArgumentParser, specials_default: int = 5) -> None:
    p.add_argument("--frames", type=int, default=1, help="number of frames F")
    p.add_argument("--patches-per-frame", type=int, default=None,
                   help="patch tokens per frame (inferred from tensor size if omitted)")
    p.add_argument("--specials-per-frame", type=int, default=specials_default,
                   help=f"special tokens per frame (default {specials_default})")
    p.add_argument("--grid", type=str, default=None, metavar="RxC", help="patch grid, e.g. 37x37")
    p.add_argument("--specials-last", action="store_true",
                   help="frames store patches first, then specials")


def _block_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--block-q", type=int, default=128, help="query block size (tokens)")
    p.add_argument("--block-k", type=int, default=64, help="key block size (tokens)")


def _grid(text):
    if text is None:
        return None
    try:
        r, c = text.lower().split("x")
        return int(r), int(c)
    except ValueError:
        raise SystemExit(f"bad --grid {text!r}, expected RxC like 37x37")


def layout_from_args(args, total_tokens: int) -> TokenLayout:
    """TokenLayout from the layout flags; patches per frame inferred from
    the token count when omitted (cli.py:61-84 semantics)."""
    f, s, p = args.frames, args.specials_per_frame, args.patches_per_frame
    if p is None:
        if total_tokens % f:
            raise SystemExit(f"{total_tokens} tokens do not divide into {f} frames")
        p = total_tokens // f - s
        if p < 1:
            raise SystemExit(f"inferred {p} patches per frame from {total_tokens} tokens, "
                             f"{f} frames, {s} specials")
    lay = TokenLayout(frames=f, patches_per_frame=p, specials_per_frame=s,
                      patch_grid=_grid(args.grid), specials_first=not args.specials_last)
    if lay.total_tokens != total_tokens:
        raise SystemExit(f"layout describes {lay.total_tokens} tokens but tensors have {total_tokens}")
    return lay


def _cmd_mask(args) -> None:
    q, k = read_tensor(args.q), read_tensor(args.k)
    if q.shape != k.shape or q.ndim != 3:
        raise SystemExit(f"q/k must share a (heads, tokens, dim) shape, got {q.shape}, {k.shape}")
    lay = layout_from_args(args, q.shape[1])
    policy = MaskPolicy(args.tau, args.rho, BlockGeometry(lay.patch_tokens, args.block_q, args.block_k))
    pidx = patch_token_indices(lay)
    mask = predict_mask(q[:, pidx], k[:, pidx], policy)
    write_mask(args.out, mask)
    if args.stats:
        w = csv.writer(sys.stdout)
        w.writerow(["head", "achieved_sparsity"])
        for h, s in enumerate(mask.achieved_sparsity()):
            w.writerow([h, _fmt(float(s))])


def _cmd_attend(args) -> None:
    q, k, v = read_tensor(args.q), read_tensor(args.k), read_tensor(args.v)
    if args.mode == "sparse" and args.mask is None:
        raise SystemExit("sparse mode requires --mask")
    inputs = AttentionInputs(q, k, v)
    if args.mode == "dense":
        write_tensor(args.out, dense_attention(inputs))
        return
    lay = layout_from_args(args, inputs.tokens)
    mask = read_mask(args.mask, BlockGeometry(lay.patch_tokens, args.block_q, args.block_k))
    job = SparseAttentionJob(inputs, lay, mask)
    if args.report:
        out, reports = sparse_attention_stats(job, panel_blocks=args.panel_blocks)
        w = csv.writer(sys.stdout)
        w.writerow(["head", "achieved_sparsity", "sparse_flops", "theoretical_speedup", "wall_ms"])
        for r in reports:
            w.writerow([r.head, _fmt(r.achieved_sparsity), r.sparse_flops,
                        _fmt(r.theoretical_speedup), _fmt(r.wall_ms)])
    else:
        out = sparse_attention(job, panel_blocks=args.panel_blocks, threads=args.threads)
    write_tensor(args.out, out)


def _cmd_bench(args) -> None:
    rows = bench_sweep(sorted(int(s) for s in args.sizes.split(",")), args.tau, args.rho,
                       repeats=args.repeats, block_q=args.block_q, block_k=args.block_k,
                       head_dim=args.dim, heads=args.heads, seed=args.seed, threads=args.threads,
                       n_matches=args.matches, dtype=args.dtype)
    write_bench_csv(args.csv if args.csv else sys.stdout, rows, with_predict=args.with_predict)


def _cmd_out_of_scope(args) -> None:
    raise SystemExit(f"'{args.command}' works on materialised attention maps or generates inputs; "
                     "it is outside the B200 data-parallel path (use the reference package)")


def _cmd_analyze(args) -> None:
    """cli.py:133-153: quadrant statistics CSV (layer, head, quadrant, mean,
    max), then per-quadrant mean/std rows over heads."""
    from .analysis import attention_quadrant_stats, quadrant_stats

    if (args.map is None) == (args.q is None):
        raise SystemExit("analyze needs either --map or --q/--k")
    if args.map is not None:
        attn_map = read_tensor(args.map)
        if attn_map.ndim == 2:
            attn_map = attn_map[None]
        layout = layout_from_args(args, attn_map.shape[1])
        stats = quadrant_stats(attn_map, layout)
    else:
        if args.k is None:
            raise SystemExit("--q needs --k")
        q, k = read_tensor(args.q), read_tensor(args.k)
        if q.ndim == 2:
            q, k = q[None], k[None]
        if q.shape != k.shape:
            raise SystemExit(f"q {q.shape} and k {k.shape} differ")
        layout = layout_from_args(args, q.shape[1])
        stats = attention_quadrant_stats(AttentionInputs(q, k, k), layout)
    out = open(args.csv, "w", newline="") if args.csv else sys.stdout
    try:
        w = csv.writer(out)
        w.writerow(["layer", "head", "quadrant", "mean", "max"])
        for quad in stats.means:
            for h in range(stats.heads):
                w.writerow([args.layer, h, quad, _fmt(stats.means[quad][h]),
                            _fmt(stats.maxes[quad][h])])
        for quad, (mm, ms, xm, xs) in stats.aggregate().items():
            w.writerow([args.layer, "mean", quad, _fmt(mm), _fmt(xm)])
            w.writerow([args.layer, "std", quad, _fmt(ms), _fmt(xs)])
    finally:
        if args.csv:
            out.close()


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="bsattn-b200",
                                 description="B200 block-sparse global attention toolkit")
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("attend", help="run dense or block-sparse attention")
    p.add_argument("--mode", choices=["dense", "sparse"], required=True)
    p.add_argument("--q", required=True)
    p.add_argument("--k", required=True)
    p.add_argument("--v", required=True)
    p.add_argument("--mask", default=None, help=".bsm block mask (sparse mode)")
    p.add_argument("--out", required=True)
    p.add_argument("--report", action="store_true",
                   help="print per-head sparsity/flops/time CSV to stdout")
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--panel-blocks", type=int, default=32,
                   help="accepted for compatibility (the kernel groups blocks itself)")
    _layout_flags(p)
    _block_flags(p)
    p.set_defaults(fn=_cmd_attend)

    p = sub.add_parser("mask", help="predict a block mask from Q and K")
    p.add_argument("--q", required=True)
    p.add_argument("--k", required=True)
    p.add_argument("--tau", type=float, required=True, help="CDF coverage threshold")
    p.add_argument("--rho", type=float, required=True, help="sparse ratio upper bound")
    p.add_argument("--out", required=True)
    p.add_argument("--stats", action="store_true",
                   help="print per-head achieved sparsity CSV to stdout")
    _layout_flags(p)
    _block_flags(p)
    p.set_defaults(fn=_cmd_mask)

    p = sub.add_parser("bench", help="dense vs sparse timing sweep")
    p.add_argument("--sizes", required=True, help="comma-separated token counts")
    p.add_argument("--tau", type=float, required=True)
    p.add_argument("--rho", type=float, required=True)
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--csv", default=None)
    p.add_argument("--dim", type=int, default=64)
    p.add_argument("--heads", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--matches", type=int, default=0,
                   help="planted matches per size (not supported: synth is out of scope)")
    p.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16")
    p.add_argument("--with-predict", action="store_true",
                   help="append the scoring-stage time (predict_ms) column")
    _block_flags(p)
    p.set_defaults(fn=_cmd_bench)

    p = sub.add_parser("analyze", help="quadrant statistics of an attention map")
    p.add_argument("--map", default=None, help=".bsat post-softmax map, (H,N,N) or (N,N)")
    p.add_argument("--q", default=None, help="(instead of --map) .bsat Q, (H,N,64)")
    p.add_argument("--k", default=None, help="(with --q) .bsat K: statistics without the map")
    p.add_argument("--csv", default=None, help="output CSV path (stdout if omitted)")
    p.add_argument("--layer", type=int, default=0, help="layer label for the CSV")
    _layout_flags(p)
    p.set_defaults(fn=_cmd_analyze)

    for name in OUT_OF_SCOPE:
        p = sub.add_parser(name, help="(out of scope in the B200 build)")
        p.add_argument("rest", nargs=argparse.REMAINDER)
        p.set_defaults(fn=_cmd_out_of_scope)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    args.fn(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
