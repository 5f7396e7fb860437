"""Minimal ``fastsum`` CLI shim (reference cli.py:162-201, 310-320): ``eval`` and
``sweep``, the subcommands the reference's acceptance gate drives (criterion 10,
test_acceptance.py:357-404).  Exit codes as the reference: 0 ok, 1 usage, 2 data.
The CLI itself is outside the B200 hot path; everything it calls is the package.
"""

import argparse
import sys

from paper_2506_02219_b200.bench import run_sweep, write_sweep_csv, write_sweep_json
from paper_2506_02219_b200.estimators import evaluate_field
from paper_2506_02219_b200.octree import build_tree
from paper_2506_02219_b200.scene_io import (GridSpec, PointsFileError, make_queries,
                                            parse_points_file, write_outputs)
from paper_2506_02219_b200.types import EstimatorConfig, KernelSpec

METHODS = {"brute": "brute_force", "brute_force": "brute_force", "bh": "barnes_hut",
           "barnes-hut": "barnes_hut", "barnes_hut": "barnes_hut", "stochastic": "stochastic",
           "telescoping": "telescoping_exhaustive",
           "telescoping_exhaustive": "telescoping_exhaustive"}
KERNELS = {"coulomb": "coulomb", "winding": "winding_dipole", "winding_dipole": "winding_dipole",
           "smooth": "smooth_exp", "smooth_exp": "smooth_exp"}


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (2 is reserved for data errors)
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(1)


def _vec3(text):
    v = tuple(float(x) for x in text.split(","))
    if len(v) != 3:
        raise argparse.ArgumentTypeError("expected x,y,z")
    return v


def _common(p):
    p.add_argument("--points", required=True)
    p.add_argument("--method", default="stochastic", choices=sorted(METHODS))
    p.add_argument("--kernel", default="coulomb", choices=sorted(KERNELS))
    p.add_argument("--alpha", type=float, default=200.0)
    p.add_argument("--beta", type=float, default=2.0)
    p.add_argument("--samples-per-subdomain", "-S", type=int, default=1)
    p.add_argument("--rr-mode", default="paper_ratio",
                   choices=["paper_ratio", "fixed_half", "disabled"])
    p.add_argument("--branching", type=int, default=None)
    p.add_argument("--max-depth", type=int, default=32)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--precision", default="f64", choices=["f32", "f64"])
    p.add_argument("--grid", type=int)
    p.add_argument("--slice")
    p.add_argument("--slice-origin", type=_vec3, default=(0.0, 0.0, 0.0))
    p.add_argument("--slice-u", type=_vec3, default=(1.0, 0.0, 0.0))
    p.add_argument("--slice-v", type=_vec3, default=(0.0, 1.0, 0.0))
    p.add_argument("--slice-extent", type=float, default=1.0)
    p.add_argument("--random-queries", type=int)
    p.add_argument("--query-seed", type=int, default=0)


def _spec(a):
    if sum(x is not None for x in (a.grid, a.slice, a.random_queries)) != 1:
        raise ValueError("pick exactly one of --grid, --slice, --random-queries")
    if a.grid is not None:
        return GridSpec("grid3d", resolution=(a.grid,) * 3)
    if a.slice is not None:
        nu, nv = (int(x) for x in a.slice.split(","))
        return GridSpec("slice_plane", resolution=(nu, nv), origin=a.slice_origin,
                        u_axis=a.slice_u, v_axis=a.slice_v, extent=a.slice_extent)
    return GridSpec("random", count=a.random_queries, seed=a.query_seed)


def _eval(a):
    kernel = KernelSpec(kind=KERNELS[a.kernel], alpha=a.alpha)
    sources = parse_points_file(a.points)
    spec = _spec(a)
    queries = make_queries(spec)
    cfg = EstimatorConfig(method=METHODS[a.method], beta=a.beta,
                          samples_per_subdomain=a.samples_per_subdomain, rr_mode=a.rr_mode,
                          seed=a.seed, branching_per_dim=a.branching, max_depth=a.max_depth,
                          precision=a.precision)
    tree = None
    if cfg.method != "brute_force":
        tree = build_tree(sources, cfg.resolved_branching, cfg.max_depth)
    result = evaluate_field(cfg, sources, kernel, queries, tree=tree)
    paths = write_outputs(result, queries, spec, a.out_prefix)
    print(f"evaluated {len(queries)} queries with {cfg.method} ({result.flagged_count} "
          f"flagged); wrote " + ", ".join(sorted(paths.values())))
    return 0


def _sweep(a):
    kernel = KernelSpec(kind=KERNELS[a.kernel], alpha=a.alpha)
    sources = parse_points_file(a.points)
    queries = make_queries(_spec(a))
    method = METHODS[a.method]
    if method not in ("barnes_hut", "stochastic"):
        raise ValueError("sweep supports barnes-hut and stochastic methods")
    if ".." in a.params:
        lo, hi = a.params.split("..", 1)
        params = [float(v) for v in range(int(lo), int(hi) + 1)]
    else:
        params = [float(v) for v in a.params.split(",")]
        if method == "stochastic":
            params = [float(int(v)) for v in params]
    records = run_sweep(sources, kernel, method, params, queries, seed=a.seed,
                        branching_per_dim=a.branching, rr_mode=a.rr_mode)
    csv_path, json_path = f"{a.out_prefix}_sweep.csv", f"{a.out_prefix}_sweep.json"
    write_sweep_csv(records, csv_path)
    write_sweep_json(json_path, {"method": method, "kernel": kernel.kind, "seed": a.seed,
                                 "params": params}, sources, kernel, queries, records)
    print(f"wrote {csv_path} and {json_path} ({len(records)} rows)")
    return 0


def main(argv=None) -> int:
    parser = _Parser(prog="fastsum", description="Fast kernel summation on B200")
    sub = parser.add_subparsers(dest="command", required=True)
    pe = sub.add_parser("eval")
    _common(pe)
    pe.add_argument("--out-prefix", default="field")
    pe.set_defaults(func=_eval)
    ps = sub.add_parser("sweep")
    _common(ps)
    ps.add_argument("--params", required=True)
    ps.add_argument("--out-prefix", default="sweep")
    ps.set_defaults(func=_sweep)
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    try:
        return args.func(args)
    except (PointsFileError, FileNotFoundError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
