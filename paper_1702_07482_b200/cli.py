"""Command line for the accelerated path (drop-in for the reference CLI's
`despeckle` and `simulate` subcommands, cli.py:20-80, 101-131).

    python -m paper_1702_07482_b200 despeckle --model M --input I --output O
    python -m paper_1702_07482_b200 simulate --input I --output O --looks L

Errors (ValueError / OSError / FloatingPointError) print `error: ...` and
exit 1 like the reference (cli.py:176-183).  Training, eval and gradcheck
are out of scope.
"""
from __future__ import annotations

import argparse
import logging
import sys

from . import io as tio
from .diffusion import run_diffusion
from .speckle import SpeckleConfig, sample_speckle, sample_speckle_gpu

log = logging.getLogger("paper_1702_07482_b200")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="paper_1702_07482_b200",
        description="B200 TNRD despeckling (GPU inference of specklediff models)")
    sub = ap.add_subparsers(dest="command", required=True)
    de = sub.add_parser("despeckle", help="run a trained model on the GPU")
    de.add_argument("--model", required=True)
    de.add_argument("--input", required=True)
    de.add_argument("--output", required=True)
    de.add_argument("--looks", type=int, default=None,
                    help="looks of the input, to warn on mismatch")
    de.add_argument("--peak", type=float, default=255.0)
    si = sub.add_parser("simulate", help="add L-look multiplicative speckle")
    si.add_argument("--input", required=True)
    si.add_argument("--output", required=True)
    si.add_argument("--looks", type=int, default=1)
    si.add_argument("--seed", type=int, default=0)
    si.add_argument("--peak", type=float, default=255.0)
    si.add_argument("--gpu", action="store_true",
                    help="draw the speckle on the GPU (same distribution, not the "
                         "reference's bit stream; tnrd_sample_speckle)")
    return ap


def _despeckle(a) -> int:
    model = tio.load_model(a.model)
    if a.looks is not None and a.looks != model.looks:
        log.warning("model trained for L=%d applied to L=%d input", model.looks, a.looks)
    out, _ = run_diffusion(tio.load_image(a.input), model)
    tio.save_image(out, a.output, peak=a.peak)
    return 0


def _simulate(a) -> int:
    sampler = sample_speckle_gpu if a.gpu else sample_speckle
    pair = sampler(tio.load_image(a.input), SpeckleConfig(looks=a.looks, seed=a.seed))
    tio.save_image(pair.noisy, a.output, peak=a.peak)
    return 0


def main(argv=None) -> int:
    logging.basicConfig(level=logging.INFO, format="%(message)s")
    a = build_parser().parse_args(argv)
    try:
        return {"despeckle": _despeckle, "simulate": _simulate}[a.command](a)
    except (ValueError, OSError, FloatingPointError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
