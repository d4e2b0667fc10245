"""Recipe: stage the UNMODIFIED reference package into oracle/_ref/ (git-ignored; it travels to
the GPU box with the snapshot like a built .so) so that bench.py's reference arm and
cpu_baseline time the reference's own CPU implementation -- microfp.quantize_rtn /
dequantize (quantizers.py:247-255, formats.py:424-442) -- instead of the numpy port.

Test/bench infrastructure only: nothing on the product path imports oracle/.  The reference is
pure Python + numpy (+ scipy in modules off this path), so "building" it is a verbatim copy
of /root/reference/pkg/src/microfp, recorded with per-file SHA-256 in oracle/_ref/SOURCE.json.
Run by __graft_entry__.build() whenever /root/reference exists (in the build container).
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/microfp"
DST = os.path.join(HERE, "_ref", "microfp")


def main() -> int:
    if not os.path.isdir(SRC):
        print(f"make_ref: {SRC} absent, keeping the existing oracle/_ref (if any)")
        return 0
    shutil.rmtree(DST, ignore_errors=True)
    os.makedirs(DST)
    files = {}
    for f in sorted(os.listdir(SRC)):
        if f.endswith(".py"):
            shutil.copy2(os.path.join(SRC, f), os.path.join(DST, f))
            files[f] = hashlib.sha256(open(os.path.join(SRC, f), "rb").read()).hexdigest()
    with open(os.path.join(HERE, "_ref", "SOURCE.json"), "w") as fh:
        json.dump({"source": SRC, "files": files}, fh, indent=1)
    print(f"make_ref: staged {len(files)} files into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
