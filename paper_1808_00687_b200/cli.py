"""Command-line front end (reference ``lsd_wfst/cli.py``).

Same subcommands, flags, output lines and exit codes as the reference's ``decode``,
``bench`` and ``lattice`` (cli.py:99-165, 200-217), with the search on the GPU:

    python -m paper_1808_00687_b200 decode --graph g.txt --posts p.txt [p2.txt ...] \\
        [--osyms syms.txt] [--mode fsd|lsd] [--beam B] [--max-active N] [--device K]
    python -m paper_1808_00687_b200 bench  --graph g.txt --posts p.txt [...] --report json
    python -m paper_1808_00687_b200 lattice --lattice-in x.lat [--lattice-beam 8]

``decode`` takes one or more posterior files and decodes them as one batch (one transcript
line per file, in order).  ``--graph`` also accepts a binary CSR cache written by
``save_wfst_binary`` (``.npz``), which skips parsing and the epsilon-cycle check; ``--save-csr``
writes one.  ``--workers`` / ``--group-size`` are accepted for compatibility and validated
like ``parallel_decode`` (parallel.py:214-217); the GPU's parallelism is the CTA.

Exit codes (cli.py:1-6): 0 success, 2 file / parse / input errors, 3 search death (the
partial result is still printed), 4 step-count invariant breach inside ``bench``.
``LSD_WFST_LOG`` sets the log level.
"""
from __future__ import annotations

import argparse
import json
import logging
import math
import os
import statistics
import sys
import time

from . import __version__
from .decoder import DecodeConfig, DecodeResult, decode_batch
from .lattice import (LatticeError, LatticeRecorder, build_lattice, lattice_best_path,
                      load_lattice, prune_lattice, save_lattice)
from .posteriors import PosteriorFormatError, classify_blank_frames, load_posteriors
from .wfst import (ParseError, SymbolError, SymbolTable, WfstError, load_wfst_binary,
                   parse_wfst_text, save_wfst_binary)

log = logging.getLogger("paper_1808_00687_b200.cli")

EXIT_OK = 0
EXIT_INPUT = 2
EXIT_SEARCH_DEAD = 3
EXIT_INVARIANT = 4

REPORT_SCHEMA = "v1"          # reference bench.py:21, report_json layout kept
DEFAULT_MODES = ("fsd-gpu", "lsd-gpu")


class StepCountViolation(AssertionError):
    """A decode reported a step count inconsistent with T - |U| (bench.py:26-27)."""


def _setup_logging() -> None:
    level = getattr(logging, os.environ.get("LSD_WFST_LOG", "WARNING").upper(), None)
    logging.basicConfig(level=level if isinstance(level, int) else logging.WARNING,
                        format="%(levelname)s %(name)s: %(message)s")


def _add_decode_args(p: argparse.ArgumentParser) -> None:
    p.add_argument("--graph", required=True, help="WFST text file, or a .npz CSR cache")
    p.add_argument("--posts", required=True, nargs="+",
                   help="posterior matrix file(s) (text or POST1 binary); several = one batch")
    p.add_argument("--isyms", help="input symbol table")
    p.add_argument("--osyms", help="output symbol table")
    p.add_argument("--mode", choices=("fsd", "lsd"), default="lsd")
    p.add_argument("--beam", type=float, default=math.inf)
    p.add_argument("--max-active", type=int, default=None)
    p.add_argument("--blank-threshold", type=float, default=0.98)
    p.add_argument("--acoustic-scale", type=float, default=1.0)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--group-size", type=int, default=32)
    p.add_argument("--strict-posteriors", action="store_true",
                   help="reject rows whose probabilities do not sum to 1")
    p.add_argument("--device", type=int, default=None, help="CUDA device index")
    p.add_argument("--save-csr", help="also write the parsed graph as a .npz CSR cache")


def _load_symbols(path):
    if path is None:
        return None
    with open(path, "r", encoding="utf-8") as fh:
        return SymbolTable.parse(fh.read())


def _load_graph(path, isyms, osyms):
    if path.endswith(".npz"):
        return load_wfst_binary(path)
    with open(path, "r", encoding="utf-8") as fh:
        return parse_wfst_text(fh.read(), isyms, osyms)


def _load_inputs(args, batch: bool = False):
    isyms, osyms = _load_symbols(args.isyms), _load_symbols(args.osyms)
    graph = _load_graph(args.graph, isyms, osyms)
    if args.save_csr:
        save_wfst_binary(graph, args.save_csr)
    if args.device is not None:
        import torch
        torch.cuda.set_device(args.device)
    if batch:   # POST1 files read natively into one page-locked table (decode consumes it)
        from .posteriors import PosteriorBatch
        posts = PosteriorBatch(args.posts, strict=args.strict_posteriors)
    else:
        posts = [load_posteriors(p, strict=args.strict_posteriors) for p in args.posts]
    if args.workers < 1:
        raise ValueError(f"workers must be >= 1, got {args.workers}")
    if args.group_size < 1:
        raise ValueError(f"group_size must be >= 1, got {args.group_size}")
    return graph, posts, osyms


def _config(args) -> DecodeConfig:
    ma = args.max_active if args.max_active and args.max_active > 0 else None
    return DecodeConfig(beam=args.beam, max_active=ma, blank_threshold=args.blank_threshold,
                        acoustic_scale=args.acoustic_scale, mode=args.mode)


def _words(labels, cost, osyms) -> str:
    out = []
    for lab in labels:
        sym = osyms.find_symbol(lab) if osyms is not None else None
        out.append(sym if sym is not None else str(lab))
    out.append(f"{cost:.4f}")
    return " ".join(out)


def cmd_decode(args) -> int:
    graph, posts, osyms = _load_inputs(args, batch=True)
    cfg = _config(args)
    recorders = [LatticeRecorder() for _ in range(len(posts))] if args.lattice_out else None
    results = decode_batch(graph, posts, cfg, mode=cfg.mode, recorder=recorders)
    code = EXIT_OK
    for i, r in enumerate(results):
        print(_words(r.olabels, r.total_cost, osyms))
        if not r.reached_final:
            log.warning("utterance %d: no token reached a final state; reporting the best "
                        "non-final token", i)
    if recorders is not None:
        for i, rec in enumerate(recorders):
            lat = build_lattice(rec, graph)
            if args.lattice_beam != math.inf:
                lat = prune_lattice(lat, args.lattice_beam)
            path = args.lattice_out if len(posts) == 1 else f"{args.lattice_out}.{i}"
            save_lattice(lat, path)
            log.info("wrote lattice with %d nodes / %d arcs to %s", lat.num_nodes,
                     lat.num_arcs, path)
    for i, r in enumerate(results):
        if r.died_at_step is not None:
            where = f"utterance {i}: " if len(results) > 1 else ""
            print(f"{where}search died at step {r.died_at_step} "
                  f"(completed {r.search_steps} steps)", file=sys.stderr)
            code = EXIT_SEARCH_DEAD
    return code


def run_bench(graph, posts, cfg: DecodeConfig, modes=DEFAULT_MODES, repeats: int = 5) -> dict:
    """Median-of-``repeats`` wall time of one batched GPU decode per mode (graph and
    posterior loading excluded; the device graph is uploaded by an untimed warm-up), with
    the reduction law steps = T - |U| asserted per utterance (bench.py:67-125)."""
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    frames = sum(p.num_frames for p in posts)
    blanks = [classify_blank_frames(p, cfg.blank_threshold).count for p in posts]
    report = {"frames": frames, "blank_frames": sum(blanks), "repeats": repeats,
              "utterances": len(posts),
              "config": {"blank_threshold": cfg.blank_threshold, "beam": cfg.beam,
                         "max_active": cfg.max_active, "acoustic_scale": cfg.acoustic_scale,
                         "device": "b200"},
              "modes": {}, "speedups": {}}
    for mode in modes:
        m = {"fsd-gpu": "fsd", "lsd-gpu": "lsd"}.get(mode)
        if m is None:
            raise ValueError(f"unknown bench mode {mode!r}")
        decode_batch(graph, posts, cfg, mode=m)          # warm-up: graph upload, workspace
        times, first = [], None
        for _ in range(repeats):
            t0 = time.perf_counter()
            res = decode_batch(graph, posts, cfg, mode=m)
            times.append(time.perf_counter() - t0)
            sig = [(r.search_steps, r.tokens_expanded) for r in res]
            if first is not None and sig != first:
                raise StepCountViolation(f"{mode}: repeated runs disagree on step/token counts")
            first = sig
        for p, b, r in zip(posts, blanks, res):
            want = p.num_frames - b if m == "lsd" else p.num_frames
            if r.died_at_step is None and r.search_steps != want:
                raise StepCountViolation(f"{mode}: search_steps={r.search_steps}, expected "
                                         f"{want} (T={p.num_frames}, |U|={b})")
        wall = statistics.median(times)
        report["modes"][mode] = {
            "search_steps": sum(r.search_steps for r in res),
            "tokens_expanded": sum(r.tokens_expanded for r in res),
            "search_wall_time_s": wall,
            "total_cost": res[0].total_cost if len(res) == 1 else [r.total_cost for r in res],
            "reached_final": (res[0].reached_final if len(res) == 1
                              else [r.reached_final for r in res]),
            "frames_per_s": frames / wall if wall > 0 else math.inf,
        }
    f, l = report["modes"].get("fsd-gpu"), report["modes"].get("lsd-gpu")
    if f and l and l["search_wall_time_s"] > 0:
        report["speedups"]["fsd-gpu/lsd-gpu"] = f["search_wall_time_s"] / l["search_wall_time_s"]
    return report


def _json_safe(v):
    if isinstance(v, float) and not math.isfinite(v):
        return repr(v)
    if isinstance(v, dict):
        return {k: _json_safe(x) for k, x in v.items()}
    if isinstance(v, list):
        return [_json_safe(x) for x in v]
    return v


def report_json(report: dict) -> str:
    return json.dumps(_json_safe({"schema": REPORT_SCHEMA, **report}), indent=2,
                      sort_keys=True) + "\n"


def report_text(report: dict) -> str:
    lines = [f"frames={report['frames']} blank_frames={report['blank_frames']} "
             f"repeats={report['repeats']} utterances={report['utterances']}",
             "config: " + " ".join(f"{k}={v}" for k, v in report["config"].items())]
    for mode, st in report["modes"].items():
        cost = st["total_cost"]
        cost = f"{cost:.4f}" if isinstance(cost, float) else f"[{len(cost)} costs]"
        fin = st["reached_final"]
        fin = ("yes" if fin else "no") if isinstance(fin, bool) else f"{sum(fin)}/{len(fin)}"
        lines.append(f"{mode:>14}: steps={st['search_steps']} tokens={st['tokens_expanded']} "
                     f"search_wall={st['search_wall_time_s']:.6f}s cost={cost} final={fin} "
                     f"frames/s={st['frames_per_s']:.0f}")
    for name, ratio in report["speedups"].items():
        lines.append(f"speedup {name}: {ratio:.2f}x")
    return "\n".join(lines) + "\n"


def cmd_bench(args) -> int:
    graph, posts, _ = _load_inputs(args)
    modes = tuple(m.strip() for m in args.modes.split(",") if m.strip())
    report = run_bench(graph, posts, _config(args), modes=modes, repeats=args.repeats)
    sys.stdout.write(report_json(report) if args.report == "json" else report_text(report))
    return EXIT_OK


def cmd_lattice(args) -> int:
    lat = load_lattice(args.lattice_in)
    if args.lattice_beam != math.inf:
        lat = prune_lattice(lat, args.lattice_beam)
    cost, olabels, _ = lattice_best_path(lat)
    print(_words(olabels, cost, _load_symbols(args.osyms)))
    if args.lattice_out:
        save_lattice(lat, args.lattice_out)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="wfst-b200",
        description="WFST Viterbi beam search on B200 GPUs with blank-frame skipping and "
                    "lattice output (drop-in for lsd-wfst's decode path).")
    parser.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("decode", help="decode one or more utterances (one GPU batch)")
    _add_decode_args(p)
    p.add_argument("--lattice-out", help="write the (optionally pruned) lattice here "
                                         "(several utterances: PATH.0, PATH.1, ...)")
    p.add_argument("--lattice-beam", type=float, default=8.0)
    p.set_defaults(func=cmd_decode)

    p = sub.add_parser("bench", help="time GPU decoding modes on one batch")
    _add_decode_args(p)
    p.add_argument("--modes", default=",".join(DEFAULT_MODES),
                   help="comma-separated: " + ",".join(DEFAULT_MODES))
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--report", choices=("text", "json"), default="text")
    p.set_defaults(func=cmd_bench)

    p = sub.add_parser("lattice", help="prune a lattice file and print its best path")
    p.add_argument("--lattice-in", required=True)
    p.add_argument("--lattice-beam", type=float, default=math.inf)
    p.add_argument("--lattice-out")
    p.add_argument("--osyms")
    p.set_defaults(func=cmd_lattice)
    return parser


def main(argv=None) -> int:
    _setup_logging()
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except StepCountViolation as exc:
        print(f"invariant breach: {exc}", file=sys.stderr)
        return EXIT_INVARIANT
    except (OSError, ParseError, SymbolError, WfstError, PosteriorFormatError, LatticeError,
            ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT


__all__ = ["main", "build_parser", "run_bench", "report_json", "report_text",
           "StepCountViolation"]
