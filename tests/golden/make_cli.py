"""MFPQ weight files written by the REAL reference CLI (``microfp quantize``, cli.py:112-153 ->
fileio.write_quant, fileio.py:138-167), for the end-to-end test of SURVEY.md 8(f) row f2:
reference CLI file -> prepare_weight(path) -> GPU quantized linear.

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli.py

Writes tests/golden/cli/: the weight / calibration tensor files the CLI generated (``microfp
gen``), and one .mfpq per command line in COMMANDS (stdout of each run in commands.txt).
"""

from __future__ import annotations

import contextlib
import io
import os

from microfp.cli import main as cli_main  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")
ROWS, COLS = 256, 1024
COMMANDS = {
    # name: quantize arguments (input weight.mfpt, output <name>.mfpq appended)
    "rtn_nvfp4_h16": ["--format", "nvfp4", "--transform", "hadamard:16"],
    "rtn_mxfp4_h32": ["--format", "mxfp4", "--transform", "hadamard:32"],
    "mrgptq_nvfp4": ["--format", "nvfp4", "--method", "mr-gptq"],                 # H16, MSE E4M3 scales, act-order
    "mrgptq_nvfp4_h128": ["--format", "nvfp4", "--method", "mr-gptq", "--transform", "hadamard:128"],
    "mrgptq_mxfp4_absmax": ["--format", "mxfp4", "--method", "mr-gptq", "--scale-opt", "absmax"],  # HW E8M0
    "mrgptq_mxfp4_fit": ["--format", "mxfp4", "--method", "mr-gptq"],             # fitted grid: GPU rejects
}


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli_main(argv)
    assert rc == 0, argv
    return buf.getvalue().strip()


def main():
    os.makedirs(HERE, exist_ok=True)
    w, calib = os.path.join(HERE, "weight.mfpt"), os.path.join(HERE, "calib.mfpt")
    log = [run(["gen", "normal", str(ROWS), str(COLS), "--seed", "11", w]),
           run(["gen", "normal", "512", str(COLS), "--seed", "12", calib])]
    for name, args in COMMANDS.items():
        extra = ["--calib", calib] if "mr-gptq" in args else []
        out = os.path.join(HERE, f"{name}.mfpq")
        log.append(f"{name}: microfp quantize weight.mfpt {name}.mfpq {' '.join(args + extra[:1] + ['calib.mfpt'] * bool(extra))}"
                   f" -> {run(['quantize', w, out] + args + extra)}")
    open(os.path.join(HERE, "commands.txt"), "w").write("\n".join(log) + "\n")
    os.remove(calib)   # only the solver needs it; the tests use the weight and the .mfpq files
    print("\n".join(log))


if __name__ == "__main__":
    main()
