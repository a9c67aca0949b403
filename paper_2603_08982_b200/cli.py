"""Command-line harness on the GPU path: the reference's `run`, `sweep` and
`verify` subcommands (cli.py:62, :119-156, :183-325) driving libsvgear through the host mirror, so
the reference's config files and QKVT tensor files work unchanged.

    python -m paper_2603_08982_b200 run    tensor.qkvt --config cfg.json [--seed S] [--policy P] [--no-timing]
    python -m paper_2603_08982_b200 sweep  tensor.qkvt --config cfg.json --density-grid 0.1,0.25,0.5
    python -m paper_2603_08982_b200 verify tensor.qkvt --config cfg.json

Same records (JSON keys, CSV header, cell order; plus one extra key, "executor", naming the GPU
executor that produced the record) and exit codes as the reference: 0 success,
1 failed verification, 2 configuration error, 3 unreadable / malformed input or unwritable output,
4 instance beyond a capability limit.  What differs, by design of this path:
  * inputs are rounded to bf16 on ingest; the executor is the tcgen05 bf16 kernel (`--executor
    bf16`, default) or the fp32 check kernel (`--executor fp32`); the config's `precision` key is
    accepted and echoed but both of its values map to a GPU executor;
  * policies on the GPU: errorAwareCompensated and topPCompensated (both budget modes).  topPDrop,
    random and oracleKnapsack are analysis baselines outside the hot path -> exit code 4; so is a
    head dimension other than 64/128;
  * the dense comparison (mapMse, outputMse) is evaluated on the device in float64 with torch — it
    is the harness's yardstick, not part of the operator.  `gen` is not provided.
There is no CPU path: without a CUDA device every subcommand fails (exit code 4).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import sys
import time

import torch

from . import _lib
from ._lib import SvgEarError
from ._tensors import ShapeError
from .analysis import build_error_table, prepare
from .attention import sparse_attend
from .config import GPU_POLICIES, POLICIES, ConfigError, RunConfig, apply_preset
from .estimator import estimate_errors_streaming
from .router import DensityBudget, relaxed_objective, route_error_aware, route_score, score_top_p
from .tensorio import TensorFormatError, read_tensor_file

DENSE_COMPARE_MAX_ENTRIES = 4_194_304  # cli.py:59
CSV_HEADER = "policy,density,relaxed_objective,map_mse,output_mse,flops,seed,c_q,c_k"
SWEEP_DEFAULT_POLICIES = ("topPCompensated", "errorAwareCompensated")


class CapabilityError(RuntimeError):
    """The instance or policy is outside what the GPU path implements (exit code 4)."""


def load_run_config(path, *, preset=None, policy=None, precision=None, seed=None) -> RunConfig:
    """RunConfig from a JSON file with the command-line overrides applied on top (preset first)."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    try:
        cfg = RunConfig.from_dict(json.loads(text))
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path} does not hold valid JSON ({exc})") from exc
    if preset:
        cfg = apply_preset(cfg, preset)
    overrides = {}
    if policy:
        overrides["policy"] = policy
    if precision:
        overrides["precision"] = precision
    if seed is not None:
        overrides["seeds"] = [seed]
    return cfg.replace(**overrides) if overrides else cfg


def _config_of(args, with_policy=True) -> RunConfig:
    return load_run_config(args.config, preset=args.preset, policy=args.policy if with_policy else None,
                           precision=args.precision, seed=getattr(args, "seed", None))


def _check_capability(q, k, v, policies, budget_mode):
    if not torch.cuda.is_available():
        raise CapabilityError("no CUDA device: this harness has no CPU path")
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ShapeError("q, k, v must be 2-D")
    if q.shape[1] != k.shape[1]:
        raise ShapeError(f"q and k head dimensions differ: {q.shape[1]} vs {k.shape[1]}")
    if v.shape[1] != k.shape[1]:
        raise CapabilityError(f"value dimension {v.shape[1]} != key dimension {k.shape[1]} (d_v == d on the GPU path)")
    if q.shape[1] not in (64, 128):
        raise CapabilityError(f"head dimension {q.shape[1]} is not 64 or 128")
    for pol in policies:
        if pol not in GPU_POLICIES:
            raise CapabilityError(f"policy {pol!r} is an analysis baseline outside the GPU hot path")


def _budget(cfg: RunConfig) -> DensityBudget:
    return DensityBudget.global_density(cfg.rho) if cfg.budget_mode == "globalDensity" else DensityBudget.top_p(cfg.p)


def _mask_for(policy, budget, prep, table):
    if policy == "errorAwareCompensated":  # cli.py:89-95
        return route_error_aware(table, budget, q_centroids=prep.q_model.centroids,
                                 k_centroids=prep.k_model.centroids)
    if budget.mode == "perClusterTopP":  # cli.py:96-104: the top-p rule itself is the mask
        return score_top_p(prep.q_model.centroids, prep.k_model.centroids, prep.q_model.sizes,
                           prep.k_model.sizes, budget.p)
    return route_score(prep.q_model.centroids, prep.k_model.centroids, prep.q_model.sizes,
                       prep.k_model.sizes, budget)


class _Dense:
    """float64 dense softmax map and output of the permuted instance (oracle.py:52-56), plus the
    map a mask implies (oracle.py:59-78); torch on the device, harness-only."""

    def __init__(self, prep):
        self.q, self.k, self.v = prep.q.double(), prep.k.double(), prep.v.double()
        self.scale = 1.0 / math.sqrt(prep.d)
        self.logits = (self.q @ self.k.T) * self.scale
        self.probs = torch.softmax(self.logits, dim=1)
        self.out = self.probs @ self.v

    def implied_map(self, prep, mask):
        km, qm = prep.k_model, prep.q_model
        kbar = torch.repeat_interleave(km.centroids.double(), km.sizes.long(), dim=0)
        comp = (self.q @ kbar.T) * self.scale
        rows = torch.repeat_interleave(torch.arange(qm.num_clusters, device=self.q.device), qm.sizes.long())
        cols = torch.repeat_interleave(torch.arange(km.num_clusters, device=self.q.device), km.sizes.long())
        entry = mask.selected.to(self.q.device)[rows][:, cols]
        return torch.softmax(torch.where(entry, self.logits, comp), dim=1)


def _evaluate(policy, prep, table, mask, dense, executor, count_table):
    dtype = torch.float32 if executor == "fp32" else torch.bfloat16
    res = sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask, dtype=dtype)
    flops = prep.q_model.flops + prep.k_model.flops + (table.flops if count_table else 0)
    flops += res.flops.exact_block + res.flops.compensation
    map_err = out_err = None
    if dense is not None:
        diff = dense.implied_map(prep, mask) - dense.probs
        map_err = float((diff * diff).mean())
        diff = res.output.double() - dense.out
        out_err = float((diff * diff).mean())
    return dict(policy=policy, density=float(mask.density), relaxed=relaxed_objective(table, mask),
                map_mse=map_err, output_mse=out_err, flops=int(flops))


def _run_single(q, k, v, cfg: RunConfig, seed, executor):
    """One seed through cluster -> estimate -> route -> attend -> compare (cli.py:119-156)."""
    prep = prepare(q, k, v, cfg.c_q, cfg.c_k, seed=seed, restarts=cfg.kmeans_restarts)
    table = build_error_table(prep, cfg.estimator_mode)
    mask = _mask_for(cfg.policy, _budget(cfg), prep, table)
    dense = _Dense(prep) if prep.n_q * prep.n_k <= DENSE_COMPARE_MAX_ENTRIES else None
    rec = _evaluate(cfg.policy, prep, table, mask, dense, executor, count_table=True)
    return {"policy": cfg.policy, "density": rec["density"], "relaxedObjective": rec["relaxed"],
            "mapMse": rec["map_mse"], "outputMse": rec["output_mse"], "flopsTotal": rec["flops"],
            "seed": seed, "clusterCounts": [prep.q_model.num_clusters, prep.k_model.num_clusters]}


def _emit(text, out_path):
    if out_path:
        with open(out_path, "w", encoding="utf-8", newline="") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def _cmd_run(args) -> int:
    cfg = _config_of(args)
    q, k, v = read_tensor_file(args.tensor)
    _check_capability(q, k, v, (cfg.policy,), cfg.budget_mode)
    lines = []
    for seed in cfg.seeds:
        t0 = time.perf_counter()
        rec = _run_single(q, k, v, cfg, seed, args.executor)
        rec["config"] = cfg.to_dict()
        rec["executor"] = args.executor
        if not args.no_timing:
            torch.cuda.synchronize()
            rec["timing"] = {"seconds": time.perf_counter() - t0}
        lines.append(json.dumps(rec))
    _emit("".join(line + "\n" for line in lines), args.out)
    return 0


def parse_density_grid(text):
    """"0.1,0.25,0.5" -> [0.1, 0.25, 0.5]; every entry a density in [0, 1]."""
    grid = []
    for piece in text.split(","):
        piece = piece.strip()
        if not piece:
            continue
        try:
            rho = float(piece)
        except ValueError as exc:
            raise ConfigError(f"density grid entry {piece!r} is not a number") from exc
        if not (0.0 <= rho <= 1.0):
            raise ConfigError(f"density grid entry {rho} lies outside [0, 1]")
        grid.append(rho)
    if not grid:
        raise ConfigError("the density grid has no entries")
    return grid


def parse_policy_list(text):
    names = tuple(piece.strip() for piece in text.split(","))
    for name in names:
        if name not in POLICIES:
            raise ConfigError(f"{name!r} is not a routing policy")
    return names


def _cmd_sweep(args) -> int:
    cfg = _config_of(args, with_policy=False)  # --policy is a comma-separated list here
    densities = parse_density_grid(args.density_grid)
    policies = parse_policy_list(args.policy) if args.policy else SWEEP_DEFAULT_POLICIES
    q, k, v = read_tensor_file(args.tensor)
    _check_capability(q, k, v, policies, "globalDensity")
    cells = {}
    for seed in cfg.seeds:  # analysis.sweep_one_seed (analysis.py:345-372): one clustering per seed
        prep = prepare(q, k, v, cfg.c_q, cfg.c_k, seed=seed, restarts=cfg.kmeans_restarts)
        table = build_error_table(prep, cfg.estimator_mode)
        dense = _Dense(prep) if prep.n_q * prep.n_k <= DENSE_COMPARE_MAX_ENTRIES else None
        for di, rho in enumerate(densities):
            for pol in policies:
                mask = _mask_for(pol, DensityBudget.global_density(rho), prep, table)
                cells[(pol, di, seed)] = _evaluate(pol, prep, table, mask, dense, args.executor,
                                                   count_table=pol == "errorAwareCompensated")
    buf = io.StringIO()
    writer = csv.writer(buf, lineterminator="\n")
    writer.writerow(CSV_HEADER.split(","))
    for pol in policies:
        for di in range(len(densities)):
            for seed in cfg.seeds:
                r = cells[(pol, di, seed)]
                writer.writerow([r["policy"], r["density"], r["relaxed"], r["map_mse"], r["output_mse"],
                                 r["flops"], seed, cfg.c_q, cfg.c_k])
    _emit(buf.getvalue(), args.out)
    return 0


def _cmd_verify(args) -> int:
    """Hard invariants of the GPU path on this instance (the reference's `verify`, cli.py:270-325,
    re-based on what can be checked without the CPU package): the tensor-core executor against the
    fp32 check executor, both against the Eq.1 mixed-logit output (attention.py:195-209) when the
    dense map fits, and the tensor-core error table against the fp32 one."""
    cfg = _config_of(args)
    q, k, v = read_tensor_file(args.tensor)
    _check_capability(q, k, v, (cfg.policy,), cfg.budget_mode)
    seed = cfg.seeds[0]
    prep = prepare(q, k, v, cfg.c_q, cfg.c_k, seed=seed, restarts=cfg.kmeans_restarts)
    table = build_error_table(prep, cfg.estimator_mode)
    mask = _mask_for(cfg.policy, _budget(cfg), prep, table)
    out16 = sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask, dtype=torch.bfloat16).output.double()
    out32 = sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask, dtype=torch.float32).output.double()
    rel = lambda a, b: float((a - b).norm() / b.norm().clamp_min(1e-300))
    checks = {"executorBf16VsFp32": {"metric": rel(out16, out32), "gate": 1e-2, "relative": True}}
    if prep.n_q * prep.n_k <= DENSE_COMPARE_MAX_ENTRIES:
        dense = _Dense(prep)
        ref = dense.implied_map(prep, mask)
        # Eq.1: exact columns weight v_j, compensated columns weight the cluster mean of v
        km = prep.k_model
        cols = torch.repeat_interleave(torch.arange(km.num_clusters, device=ref.device), km.sizes.long())
        vbar = torch.zeros(km.num_clusters, prep.d, dtype=torch.float64, device=ref.device).index_add_(0, cols, dense.v)
        vbar = (vbar / km.sizes.double().unsqueeze(1))[cols]
        rows = torch.repeat_interleave(torch.arange(prep.q_model.num_clusters, device=ref.device), prep.q_model.sizes.long())
        entry = mask.selected.to(ref.device)[rows][:, cols]
        want = (ref * entry) @ dense.v + (ref * ~entry) @ vbar
        checks["executorReference"] = {"metric": rel(out32, want), "gate": 1e-4, "relative": True}
    if cfg.estimator_mode == "valueAware":
        t32 = estimate_errors_streaming(prep.q_model, prep.k_model, prep.k, prep.v, fp32_check=True)
        denom = max(1.0, float(t32.error_sum.abs().max()))
        checks["estimatorTensorVsFp32"] = {"metric": float((table.error_sum - t32.error_sum).abs().max()) / denom,
                                           "gate": 1e-3}
    for c in checks.values():
        c["pass"] = c["metric"] <= c["gate"]
    ok = all(c["pass"] for c in checks.values())
    report = {"checks": checks, "density": float(mask.density), "pass": ok}
    _emit(json.dumps(report, indent=2) + "\n", args.out)
    return 0 if ok else 1


# (flag, argparse keywords) shared by every subcommand
_COMMON_FLAGS = (
    ("--config", dict(required=True, help="RunConfig JSON path")),
    ("--preset", dict(choices=["paper"], help="apply a named configuration preset")),
    ("--seed", dict(type=int, help="run this one seed instead of the config's seed list")),
    ("--policy", dict(help="routing policy (a comma-separated list for sweep)")),
    ("--precision", dict(choices=["double", "single-executor"],
                         help="accepted for compatibility with the reference and echoed; see --executor")),
    ("--executor", dict(choices=["bf16", "fp32"], default="bf16",
                        help="GPU executor: tcgen05 bf16 (default) or the fp32 check kernel")),
    ("--no-timing", dict(action="store_true", help="leave the timing field out (byte-stable output)")),
    ("--out", dict(help="write the output to this file instead of stdout")),
)
_SUBCOMMANDS = {
    "run": ("one JSON line per seed", _cmd_run, ()),
    "sweep": ("policy x density x seed grid as CSV", _cmd_sweep,
              (("--density-grid", dict(required=True, help="comma-separated densities, e.g. 0.1,0.25,0.5")),
               ("--workers", dict(type=int, help="accepted for compatibility; seeds run on one device")))),
    "verify": ("invariant checks of the GPU path, JSON report", _cmd_verify, ()),
}
# exception type -> (stderr label, exit code); checked in order (ConfigError and ShapeError are ValueErrors)
_EXIT_CODES = (
    (ConfigError, "config error", 2),
    ((TensorFormatError, ShapeError), "input error", 3),
    (OSError, "io error", 3),
    (CapabilityError, "capability error", 4),
)
# libsvgear statuses that ARE capability limits (shape / policy the kernels do not implement, or no
# device at all); the others (bad argument, workspace, a failed CUDA call on a working device) are
# bugs or runtime faults and propagate with a traceback instead of being reported as a limit
_CAPABILITY_STATUSES = (_lib.ESHAPE, _lib.EUNSUPPORTED)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2603_08982_b200", description="SVG-EAR attention harness (B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (summary, _, extra) in _SUBCOMMANDS.items():
        p = sub.add_parser(name, help=summary)
        p.add_argument("tensor", help="QKVT tensor file to read")
        for flag, kw in extra + _COMMON_FLAGS:
            p.add_argument(flag, **kw)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    handler = _SUBCOMMANDS[args.command][1]
    try:
        return handler(args)
    except Exception as exc:  # noqa: BLE001 - mapped to the documented exit codes, anything else propagates
        if isinstance(exc, SvgEarError) and exc.status in _CAPABILITY_STATUSES:
            print(f"capability error: {exc}", file=sys.stderr)
            return 4
        for kinds, label, code in _EXIT_CODES:
            if isinstance(exc, kinds):
                print(f"{label}: {exc}", file=sys.stderr)
                return code
        raise


if __name__ == "__main__":
    sys.exit(main())
