"""``python -m paper_2201_05024_b200.cli`` -- the file-driven train / detect
commands of the reference CLI (kapsm/cli.py:168-198) on the GPU path.

    train  --iq CAPTURE --pilots SYMBOLS --out MODEL [--window W --epsilon E
           --w-l --w-g --sigma-sq --precision f64|f32]
    detect MODEL CAPTURE OUT [--precision f32|f64]
    bench  [--dict-sizes ... --batch-sizes ... --stages ... --workers ...
           --repeats R --seed S --antennas M --precision --json --out FILE]

``bench`` is the reference's ``kapsm bench`` (cli.py:144-165): the detection
harness (bench.py here) with B200 rows, CSV or JSON on stdout / --out, exit 1
when a row fails the checksum gate.

Training runs the persistent GPU trainer on the first len(pilots) samples of
the capture; detection runs the GPU evaluation engine and writes float32
(I, Q) estimates.  The reference reads its APSM/engine settings from an INI
run configuration (out of scope here); they are flags instead.
Exit codes as cli.py:252-262: 0 ok, 2 usage / file format / missing file,
1 any other error.
"""

from __future__ import annotations

import argparse
import sys

from .apsm import ApsmConfig, train
from .bench import bench_detection, report_to_csv, report_to_json
from .engine import EngineConfig, batch_detect
from .kernels import KernelParams, zero_filter
from .modelio import FileFormatError, load_iq, load_model, load_symbols, save_model, save_symbols


def _train(a) -> int:
    rx = load_iq(a.iq)
    pil = load_symbols(a.pilots)
    if pil.size == 0:
        raise FileFormatError(f"{a.pilots}: the pilot stream is empty; nothing to train on")
    if pil.size > rx.shape[0]:
        raise FileFormatError(f"{a.pilots}: {pil.size} pilot symbols but only {rx.shape[0]} "
                              f"samples in {a.iq}")
    params = KernelParams(a.w_l, a.w_g, a.sigma_sq)
    cfg = ApsmConfig(window=a.window, epsilon=a.epsilon, params=params)
    f = train(zero_filter(2 * rx.shape[1]), zip(rx[:pil.size], pil), cfg, precision=a.precision)
    save_model(a.out, f, params)
    print(f"trained {f.n_atoms} atoms from {pil.size} pilots -> {a.out}", file=sys.stderr)
    return 0


def _detect(a) -> int:
    f, params = load_model(a.model)
    rx = load_iq(a.iq)
    if 2 * rx.shape[1] != f.dim:
        raise FileFormatError(f"{a.iq}: the capture has {rx.shape[1]} antennas, the model "
                              f"expects {f.dim // 2}")
    save_symbols(a.out, batch_detect(f, rx, params, EngineConfig(precision=a.precision)))
    return 0


def _bench(a) -> int:
    rep = bench_detection(a.dict_sizes, a.batch_sizes, a.stages, a.workers, a.repeats,
                          seed=a.seed, antennas=a.antennas,
                          params=KernelParams(a.w_l, a.w_g, a.sigma_sq),
                          engine_template=EngineConfig(precision=a.precision))
    text = report_to_json(rep) if a.json else report_to_csv(rep)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    if rep.has_failures:
        bad = sorted({r.stage for r in rep.rows if not r.ok})
        print(f"error: checksum mismatch against baseline for stage(s): {', '.join(bad)}",
              file=sys.stderr)
        return 1
    return 0


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="kapsm_b200",
                                 description="APSM multiuser detector on B200: file-based "
                                             "train / detect")
    sub = ap.add_subparsers(dest="command", required=True)
    t = sub.add_parser("train", help="train a model from a capture and its known pilots")
    t.add_argument("--iq", required=True)
    t.add_argument("--pilots", required=True, help="pilot symbols (raw float32 I, Q pairs)")
    t.add_argument("--out", required=True)
    t.add_argument("--window", type=int, default=20)
    t.add_argument("--epsilon", type=float, default=0.01)
    t.add_argument("--w-l", type=float, default=0.5)
    t.add_argument("--w-g", type=float, default=0.5)
    t.add_argument("--sigma-sq", type=float, default=0.05)
    t.add_argument("--precision", choices=("f64", "f32"), default="f64")
    t.set_defaults(func=_train)
    d = sub.add_parser("detect", help="detect the symbols of a capture with a trained model")
    d.add_argument("model")
    d.add_argument("iq")
    d.add_argument("out")
    d.add_argument("--precision", choices=("f64", "f32"), default="f64")
    d.set_defaults(func=_detect)
    b = sub.add_parser("bench", help="detection latency harness (checksum-gated rows)")
    b.add_argument("--dict-sizes", type=int, nargs="+", default=[10_000])
    b.add_argument("--batch-sizes", type=int, nargs="+", default=[4_096])
    b.add_argument("--stages", nargs="+", default=["baseline", "tiled", "balanced"])
    b.add_argument("--workers", type=int, nargs="+", default=[1])
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--antennas", type=int, default=16)
    b.add_argument("--w-l", type=float, default=0.5)
    b.add_argument("--w-g", type=float, default=0.5)
    b.add_argument("--sigma-sq", type=float, default=0.05)
    b.add_argument("--precision", choices=("f64", "f32"), default="f64")
    b.add_argument("--json", action="store_true")
    b.add_argument("--out")
    b.set_defaults(func=_bench)
    return ap


def main(argv=None) -> int:
    try:
        a = _parser().parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 2
    try:
        return a.func(a)
    except (FileFormatError, FileNotFoundError, IsADirectoryError, PermissionError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except Exception as exc:  # noqa: BLE001 -- the CLI boundary maps everything else to 1
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
