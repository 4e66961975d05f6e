"""Detection benchmark harness with B200 rows (mirror of kapsm/bench.py).

Same API, row schema and "no timing without a passing checksum" rule as the
reference harness (pkg/src/kapsm/bench.py:36-201): for every (dictionary size,
batch size) cell one synthetic problem is drawn with the reference's
distribution and seeding (bench.py:81-98, ``default_rng([seed, dict_size,
batch_size])``), a reference output is computed, and each requested (stage,
workers) combination is timed over ``repeats`` calls of ``batch_detect``.

On the B200 there is one detection path (engine.py here): ``stage`` and
``workers`` label the rows of the reference's grid but select the same CUDA
kernels.  The reference output of a cell (the role of the reference's
"baseline" stage, which evaluates by explicit differences) is the GPU
evaluation kernel at the template's precision -- explicit differences too,
no norm expansion.  A row's timing is the wall clock of the public
``batch_detect`` call (host -> device copy, kernel, device -> host copy), as
the reference times its own call; throughput counts realified kernel
evaluations (two per complex detection, bench.py:185).
"""

from __future__ import annotations

import hashlib
import json
import time
from dataclasses import asdict, dataclass
from typing import Optional, Sequence

import numpy as np

from .engine import STAGES, EngineConfig, batch_detect, batch_evaluate
from .kernels import FilterState, KernelParams

__all__ = ["BenchRow", "BenchReport", "bench_detection", "report_to_csv", "report_to_json",
           "CSV_COLUMNS"]

CSV_COLUMNS = ("stage", "dict_size", "batch_size", "workers", "median_us", "p95_us",
               "throughput_evals_per_s", "checksum", "ok")


@dataclass(frozen=True)
class BenchRow:
    """One (stage, dict_size, batch_size, workers) cell; timings NaN when the
    checksum gate failed (bench.py:49-67)."""

    stage: str
    dict_size: int
    batch_size: int
    workers: int
    median_us: float
    p95_us: float
    throughput_evals_per_s: float
    checksum: str
    ok: bool


@dataclass(frozen=True)
class BenchReport:
    rows: tuple

    @property
    def has_failures(self) -> bool:
        return any(not r.ok for r in self.rows)


def _sha(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest()


def synthetic_problem(dict_size: int, batch_size: int, antennas: int, params: KernelParams,
                      rng: np.random.Generator):
    """Random filter + complex inputs with live Gaussian terms: entries scaled
    so squared distances sit near 2 sigma^2 (bench.py:81-98, same draws in the
    same order, so a seed gives the reference's problem)."""
    dim = 2 * antennas
    s = np.sqrt(params.sigma_sq / dim)
    atoms = s * rng.standard_normal((dict_size, dim))
    coeffs = rng.standard_normal(dict_size) / np.sqrt(dict_size)
    theta = rng.standard_normal(dim)
    re = rng.standard_normal((batch_size, antennas))
    im = rng.standard_normal((batch_size, antennas))
    return FilterState(theta, atoms, coeffs), s * (re + 1j * im)


def _reference_output(f: FilterState, inputs: np.ndarray, params: KernelParams, prec: str):
    """The cell's reference: the explicit-difference evaluation kernel on the
    realified inputs, recombined as g = f(r1) + i f(r2)."""
    r1 = np.hstack([inputs.real, inputs.imag])
    r2 = np.hstack([inputs.imag, -inputs.real])
    y = batch_evaluate(f, np.vstack([r1, r2]), params, EngineConfig(precision=prec))
    n = inputs.shape[0]
    return y[:n] + 1j * y[n:]


def _max_rel(out: np.ndarray, ref: np.ndarray) -> float:
    d = float(np.max(np.abs(ref)))
    diff = float(np.max(np.abs(out - ref), initial=0.0))
    return diff / d if d else diff


def bench_detection(dict_sizes: Sequence[int], batch_sizes: Sequence[int],
                    stages: Sequence[str] = STAGES, workers: Sequence[int] = (1,),
                    repeats: int = 5, seed: int = 0, antennas: int = 16,
                    params: Optional[KernelParams] = None,
                    engine_template: Optional[EngineConfig] = None,
                    corrupt_stage: Optional[str] = None) -> BenchReport:
    """Time B200 detection over the (dict, batch, stage, workers) grid
    (bench.py:108-201): gate first (1e-9 relative in f64, 1e-4 in f32), then
    median / p95 wall time of ``repeats`` calls after one warm-up call.
    ``corrupt_stage`` perturbs that stage's outputs before the gate (the
    reference's hook for exercising the failure path)."""
    if repeats < 5:
        raise ValueError(f"repeats must be >= 5 for stable medians, got {repeats}")
    for st in stages:
        if st not in STAGES:
            raise ValueError(f"unknown stage {st!r}; expected one of {STAGES}")
    params = KernelParams() if params is None else params
    tmpl = EngineConfig() if engine_template is None else engine_template
    tol = 1e-4 if tmpl.precision == "f32" else 1e-9
    rows = []
    for dsz in dict_sizes:
        for bsz in batch_sizes:
            f, inputs = synthetic_problem(dsz, bsz, antennas, params,
                                          np.random.default_rng([seed, dsz, bsz]))
            ref = _reference_output(f, inputs, params, tmpl.precision)
            ref_sum = _sha(ref)
            for st in stages:
                for nw in workers:
                    cfg = EngineConfig(stage=st, tile_atoms=tmpl.tile_atoms,
                                       tile_inputs=tmpl.tile_inputs, chunk_dim=tmpl.chunk_dim,
                                       workers=nw,
                                       deterministic_reduction=tmpl.deterministic_reduction,
                                       precision=tmpl.precision)
                    out = batch_detect(f, inputs, params, cfg)          # warm-up
                    ts = []
                    for _ in range(repeats):
                        t0 = time.perf_counter()
                        out = batch_detect(f, inputs, params, cfg)
                        ts.append(time.perf_counter() - t0)
                    if st == corrupt_stage:
                        out = out + (1.0 + 1.0j)
                    if _max_rel(out, ref) <= tol:
                        med = float(np.median(ts))
                        rows.append(BenchRow(st, dsz, bsz, nw, med * 1e6,
                                             float(np.percentile(ts, 95)) * 1e6,
                                             2.0 * bsz / med, ref_sum, True))
                    else:
                        nan = float("nan")
                        rows.append(BenchRow(st, dsz, bsz, nw, nan, nan, nan, _sha(out), False))
    return BenchReport(tuple(rows))


def _csv_cell(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return "" if np.isnan(v) else repr(v)
    return str(v)


def report_to_csv(report: BenchReport) -> str:
    """CSV in the reference column order; failed timings are empty cells."""
    out = [",".join(CSV_COLUMNS)]
    for r in report.rows:
        d = asdict(r)
        out.append(",".join(_csv_cell(d[c]) for c in CSV_COLUMNS))
    return "\n".join(out) + "\n"


def report_to_json(report: BenchReport) -> str:
    """{"rows": [...]} with failed timings as null (bench.py:219-228)."""
    rows = []
    for r in report.rows:
        d = asdict(r)
        for k in ("median_us", "p95_us", "throughput_evals_per_s"):
            if np.isnan(d[k]):
                d[k] = None
        rows.append(d)
    return json.dumps({"rows": rows}, indent=2) + "\n"
