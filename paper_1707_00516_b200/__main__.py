"""``python -m paper_1707_00516_b200`` -- the reference CLI's comparison path on the B200.

Mirrors ``fastid compare`` (cli.py:66-92, 196-209) for the parts on the hot
path: panel files in (native ingest, ingest.py), the score matrix out in the
reference's CSV or packed-binary format, exit codes 0 / 1 (invalid input) /
2 (usage).  ``search`` adds the fused top-k for database-scale jobs.  The
reference's budget / tile / worker / ledger options belong to its CPU
scheduler and are not offered.
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np

EXIT_OK, EXIT_INPUT = 0, 1


def _write_csv(path, ref_ids, query_ids, scores: np.ndarray) -> None:
    # io.py:160-166 / _csv_data_rows: "ref_id,<query ids>" then "<ref id>,<cells>" rows
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("ref_id," + ",".join(query_ids) + "\n")
        for rid, row in zip(ref_ids, scores):
            fh.write(rid + "," + ",".join(map(str, row.tolist())) + "\n")


def cmd_compare(args) -> int:
    from . import compare_b200, compare_to_fidm
    from .ingest import load_panel

    t0 = time.perf_counter()
    refs = load_panel(args.refs, args.word_width)
    queries = load_panel(args.queries, args.word_width)
    t1 = time.perf_counter()
    if args.format == "binary":
        compare_to_fidm(refs, queries, args.out, args.formulation)
    else:
        m = compare_b200(refs, queries, args.formulation)
        _write_csv(args.out, m.ref_ids, m.query_ids, m.scores)
    t2 = time.perf_counter()
    print(f"compared {refs.n_profiles} refs x {queries.n_profiles} queries on the B200; "
          f"load {1e3 * (t1 - t0):.1f} ms, compare+write {1e3 * (t2 - t1):.1f} ms")
    print(f"scores written to {args.out}")
    return EXIT_OK


def cmd_search(args) -> int:
    from . import topk
    from .ingest import load_panel

    refs = load_panel(args.refs, args.word_width)
    queries = load_panel(args.queries, args.word_width)
    res = topk(refs, queries, args.k, args.max_score, args.formulation)
    with open(args.out, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("query_id,rank,ref_id,score\n")
        for j, qid in enumerate(res.query_ids):
            for r in range(args.k):
                x = int(res.index[j, r])
                if x < 0:
                    break
                fh.write(f"{qid},{r + 1},{refs.ids[x]},{int(res.scores[j, r])}\n")
    print(f"top-{args.k} of {refs.n_profiles} refs for {queries.n_profiles} queries written to {args.out}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_1707_00516_b200",
                                description="FastID AND-NOT/popcount comparison on the B200.")
    sub = p.add_subparsers(dest="command", required=True)
    c = sub.add_parser("compare", help="score a reference panel against a query panel (full matrix)")
    c.add_argument("--refs", required=True)
    c.add_argument("--queries", required=True)
    c.add_argument("--out", required=True)
    c.add_argument("--format", choices=("csv", "binary"), default="csv")
    c.add_argument("--word-width", type=int, choices=(32, 64), default=64)
    c.add_argument("--formulation", choices=("auto", "tensor_f4", "tensor_i8", "popc"), default="auto")
    c.set_defaults(func=cmd_compare)
    s = sub.add_parser("search", help="per query, the k closest references (score asc, index asc)")
    s.add_argument("--refs", required=True)
    s.add_argument("--queries", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("-k", type=int, default=16)
    s.add_argument("--max-score", type=int, default=None)
    s.add_argument("--word-width", type=int, choices=(32, 64), default=64)
    s.add_argument("--formulation", choices=("auto", "tensor_f4", "tensor_i8", "popc"), default="auto")
    s.set_defaults(func=cmd_search)
    return p


def main(argv=None) -> int:
    from .errors import FastIdError

    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (FastIdError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
