"""Experiment-harness hook: run the reference's Newton settings on the GPU solver
and write the reference's trace / summary CSVs.

The reference's harness (bench.py:36-46, 158-179, 243-330) drives
`newton_solve` through `execute_run(prob, test_set, run)` and writes one trace
CSV per run plus `summary.csv`.  This module provides:

  * SUMMARY_COLUMNS / RunResult / write_summary_csv -- the summary schema and
    writer of bench.py:36-46, 112-119, 243-267 (byte-identical output; the only
    timing column is time_to_target_seconds);
  * execute_run -- bench.py:158-179 for the Newton methods, running the GPU
    `newton_solve` with the reference's configs; `make_execute_run(fallback)`
    returns a drop-in replacement for the reference's `execute_run` that sends
    every other method (the first-order baselines, out of scope here) to
    `fallback` (INTEGRATION.md shows the one-line patch);
  * run_experiment -- bench.py:270-330 for specs whose solvers are all Newton
    methods (or with a `first_order` delegate): load, normalise and split on the
    device, run, write the CSVs.  Figures are the reference's plotting code and
    stay out of scope (`figures` is ignored).
"""

import csv
import os
from dataclasses import dataclass, field

from .cg import CgConfig
from .data import normalize_columns, train_test_split
from .errors import DataError
from .io import load_csv, load_libsvm
from .linesearch import LineSearchConfig
from .newton import NewtonConfig, make_variant, newton_solve
from .sampling import SampleConfig
from .softmax import SoftmaxProblem
from .trace import SolveTrace, format_float, write_trace_csv

# CLI method name -> newton variant name (bench.py:28-32)
NEWTON_METHODS = {
    "full-newton": "full",
    "subnewton-100": "subsampled-100",
    "subnewton-20": "subsampled-20",
}

SUMMARY_COLUMNS = (  # bench.py:36-46
    "solver",
    "method",
    "learning_rate",
    "iterations",
    "final_objective",
    "best_test_acc",
    "time_to_target_seconds",
    "classification",
    "termination",
)


@dataclass
class RunResult:
    """bench.py:112-119 (learning_rate is None for the Newton variants)."""

    label: str
    method: str
    learning_rate: float
    trace: SolveTrace
    trace_path: str = ""
    classification: str = ""


@dataclass
class ExperimentResult:
    """bench.py:122-127."""

    runs: list
    summary_path: str
    figure_paths: list = field(default_factory=list)
    lipschitz: float = None


def _format_lr(lr):
    return f"{lr:.6g}"


def _summary_row(result, target):
    """bench.py:247-260."""
    trace = result.trace
    tta = ""
    if target is not None:
        t = trace.time_to_accuracy(target)
        tta = format_float(t) if t is not None else ""
    return [
        result.label,
        result.method,
        _format_lr(result.learning_rate) if result.learning_rate is not None else "",
        str(trace.iterations),
        format_float(trace.final_objective),
        format_float(trace.best_test_acc),
        tta,
        result.classification,
        trace.reason,
    ]


def write_summary_csv(path, results, target_accuracy=None):
    """bench.py:262-267: header row then one row per result, '\\n' line ends."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        writer = csv.writer(fh, lineterminator="\n")
        writer.writerow(SUMMARY_COLUMNS)
        for result in results:
            writer.writerow(_summary_row(result, target_accuracy))


def newton_config(run):
    """The NewtonConfig bench.py:161-171 builds from a SolverRun (duck-typed:
    method, epochs, epsilon, cg_tol, cg_max_iters, seed)."""
    return make_variant(
        NEWTON_METHODS[run.method],
        NewtonConfig(
            epsilon=run.epsilon,
            max_outer_iters=run.epochs,
            cg=CgConfig(theta=run.cg_tol, max_iters=run.cg_max_iters),
            ls=LineSearchConfig(),
            samples=SampleConfig(seed=run.seed),
        ),
    )


def execute_run(prob, test_set, run, learning_rate=None):
    """bench.py:158-171 for a Newton method, on the GPU solver."""
    if run.method not in NEWTON_METHODS:
        raise ValueError(f"{run.method!r} is not a Newton method; the GPU path runs "
                         f"{sorted(NEWTON_METHODS)} (use make_execute_run(fallback))")
    return newton_solve(prob, newton_config(run), test_set=test_set, solver_name=run.method)


def make_execute_run(fallback):
    """A drop-in for the reference's execute_run: Newton methods on the GPU,
    anything else through `fallback` (the reference's own function)."""

    def run_any(prob, test_set, run, learning_rate=None):
        if run.method in NEWTON_METHODS:
            return execute_run(prob, test_set, run)
        return fallback(prob, test_set, run, learning_rate=learning_rate)

    return run_any


def load_dataset(path, fmt, n_classes, n_features=None):
    """bench.py:141-146."""
    if fmt == "libsvm":
        return load_libsvm(path, n_classes, n_features=n_features)
    if fmt == "csv":
        return load_csv(path, n_classes)
    raise ValueError(f"unknown dataset format {fmt!r}; expected libsvm or csv")


def prepare_data(spec):
    """bench.py:149-155: load, optionally normalise, split -- on the device."""
    ds = load_dataset(spec.dataset_path, spec.fmt, spec.n_classes, spec.n_features)
    if spec.normalize:
        ds = normalize_columns(ds)
    return train_test_split(ds, spec.split_fraction, spec.seed)


def run_experiment(spec, first_order=None):
    """bench.py:270-311 for the reference's ExperimentSpec (duck-typed): every
    Newton setting runs on the GPU; other settings go to `first_order(prob,
    test, run) -> list of RunResult` (e.g. a wrapper around the reference's
    sweep code) or raise.  Writes trace_<label>.csv per run and summary.csv."""
    if not spec.solvers:
        raise ValueError("experiment spec needs at least one solver")
    if spec.lam < 0:
        raise DataError("lambda must be >= 0")
    train, test = prepare_data(spec)
    prob = SoftmaxProblem(train, spec.lam)
    results = []
    for run in spec.solvers:
        if run.method in NEWTON_METHODS:
            results.append(RunResult(run.method, run.method, None,
                                     execute_run(prob, test, run)))
        elif first_order is not None:
            results.extend(first_order(prob, test, run))
        else:
            raise ValueError(f"{run.method!r}: first-order baselines are outside the GPU "
                             "path; pass first_order=...")
    os.makedirs(spec.out_dir, exist_ok=True)
    for result in results:
        result.trace_path = os.path.join(spec.out_dir, f"trace_{result.label}.csv")
        write_trace_csv(result.trace_path, result.trace.records)
    summary_path = os.path.join(spec.out_dir, "summary.csv")
    write_summary_csv(summary_path, results, spec.target_accuracy)
    return ExperimentResult(results, summary_path)


__all__ = ["NEWTON_METHODS", "SUMMARY_COLUMNS", "RunResult", "ExperimentResult",
           "write_summary_csv", "newton_config", "execute_run", "make_execute_run",
           "load_dataset", "prepare_data", "run_experiment"]
