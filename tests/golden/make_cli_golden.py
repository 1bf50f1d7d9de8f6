"""Generate CLI report fixtures by running the REFERENCE command line itself.

Run in the build container (the reference is only mounted here):

    python tests/golden/make_cli_golden.py

For each case below it writes a seeded matrix as PODM (with the reference's
own writer), runs ``python -m podsketch run ...`` from /root/reference/pkg/src
in a subprocess, and stores the JSON report the reference printed, minus its
wall-clock fields, in ``cli_reports.json`` next to this script.
``tests/test_gpu_cli.py::test_report_matches_reference_cli`` replays the same
command lines through the drop-in's CLI and compares the reports field by
field (reference cli.py / reporting.py: config echo, sigma, traces, passes,
angles and the Wedin block).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

# (name, argv after "run"; MATRIX is substituted by the PODM path)
CASES = [
    ("isma_l2n", ["isma", "MATRIX", "--k", "3", "--seed", "4", "--c", "12", "--tau", "0.999"]),
    ("isma_unf_subspace", ["isma", "MATRIX", "--k", "3", "--seed", "5", "--c", "10",
                           "--strategy", "unf", "--criterion", "subspace", "--tau", "0.99"]),
    ("isma_ls_rows_ref", ["isma", "MATRIX", "--k", "3", "--seed", "6", "--c", "12", "--w", "40",
                          "--strategy", "ls", "--rows", "--reference", "MATRIX"]),
    ("isma_ort_nofinal", ["isma", "MATRIX", "--k", "4", "--seed", "2", "--c", "10",
                          "--strategy", "ort", "--no-finalize"]),
    ("gram_ref", ["gram", "MATRIX", "--k", "3", "--reference", "MATRIX"]),
    ("ltsvd", ["ltsvd", "MATRIX", "--k", "3", "--seed", "9", "--c", "30"]),
    ("ctsvd", ["ctsvd", "MATRIX", "--k", "3", "--seed", "9", "--c", "30"]),
    ("incremental", ["incremental", "MATRIX", "--k", "3", "--seed", "1", "--blocks", "4",
                     "--c", "8"]),
]


def case_matrix():
    """80 x 50, rank 4 plus noise: the matrix of tests/test_gpu_cli.py's fixture."""
    rng = np.random.default_rng(909)
    u = np.linalg.qr(rng.standard_normal((80, 4)))[0]
    v = np.linalg.qr(rng.standard_normal((50, 4)))[0]
    a = (u * np.array([10.0, 7.0, 4.0, 2.0])) @ v.T
    return a + 0.05 * rng.standard_normal((80, 50))


def strip_timing(rep):
    rep = json.loads(json.dumps(rep))
    rep.pop("timing", None)
    for t in rep.get("traces", []):
        t.pop("wall_time", None)
    return rep


def main():
    sys.path.insert(0, REF_SRC)
    import podsketch  # the reference

    out = {"matrix": "case_matrix() of tests/golden/make_cli_golden.py", "cases": {}}
    env = dict(os.environ, PYTHONPATH=REF_SRC)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "d.podm")
        podsketch.write_matrix(path, case_matrix())
        for name, argv in CASES:
            args = [path if x == "MATRIX" else x for x in argv]
            p = subprocess.run([sys.executable, "-m", "podsketch", "run"] + args, env=env,
                               capture_output=True, text=True, cwd=d)
            assert p.returncode == 0, (name, p.stderr)
            rep = strip_timing(json.loads(p.stdout))
            # the echoed matrix path is machine-specific
            out["cases"][name] = {"argv": argv, "report": rep}
    with open(os.path.join(HERE, "cli_reports.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"wrote {len(out['cases'])} reference CLI reports")


if __name__ == "__main__":
    main()
