"""Stage the reference package's own test suite for a run against the drop-in.

The reference's tests (``/root/reference/pkg/tests``) are copied, unmodified,
into ``tests/reference_suite/_staged/`` -- a git-ignored directory (the
reference's sources never enter this repository's history) that travels to
the GPU box with the working tree, like the built ``.so``.  The sibling
``conftest.py`` aliases ``podsketch`` to ``paper_1905_05107_b200`` so those
files import the drop-in instead of the reference, and marks every staged
test ``gpu`` (the drop-in computes on the device only).

Run by ``__graft_entry__.build()`` when /root/reference is present, or by hand:
``python tests/reference_suite/stage.py``.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_staged")


def stage(src=SRC, dst=DST):
    if not os.path.isdir(src):
        return False
    os.makedirs(dst, exist_ok=True)
    manifest = []
    for name in sorted(os.listdir(src)):
        if not name.endswith(".py"):
            continue
        shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
        with open(os.path.join(dst, name), "rb") as f:
            manifest.append(f"{hashlib.sha256(f.read()).hexdigest()[:16]}  {name}")
    with open(os.path.join(dst, "MANIFEST"), "w") as f:
        f.write("\n".join(manifest) + "\n")
    return True


if __name__ == "__main__":
    ok = stage()
    print("staged" if ok else f"{SRC} absent: nothing staged", file=sys.stderr)
