"""CLI runs on the GPU (reference cli.py semantics): every algorithm emits a
schema-valid report, seeded runs repeat exactly minus timing, references add
angles and the Wedin block, factors round-trip through PODF, and the exit
codes of the reference."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
from podtest_util import make_low_rank

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import cli, reporting  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture
def mat(tmp_path):
    rng = np.random.default_rng(909)
    a = make_low_rank(80, 50, 4, rng) + 0.05 * rng.standard_normal((80, 50))
    p = str(tmp_path / "d.podm")
    pod.write_matrix(p, a)
    return p, a


def _run(capsys, *argv):
    assert cli.main(list(argv)) == 0
    rep = json.loads(capsys.readouterr().out)
    reporting.validate_report(rep)
    return rep


def _strip(rep):
    rep = json.loads(json.dumps(rep))
    rep.pop("timing")
    for t in rep["traces"]:
        t.pop("wall_time")
    return rep


@pytest.mark.parametrize("alg", ["gram", "ltsvd", "ctsvd", "isma", "incremental"])
def test_every_algorithm_reports(capsys, mat, alg):
    path, a = mat
    rep = _run(capsys, "run", alg, path, "--k", "3", "--seed", "4")
    assert rep["config"]["algorithm"] == alg and len(rep["sigma"]) == 3
    assert (rep["traces"] != []) == (alg in ("isma", "incremental"))
    assert rep["passes"] >= 1
    s = np.linalg.svd(a, compute_uv=False)
    if alg == "gram":
        np.testing.assert_allclose(rep["sigma"], s[:3], rtol=1e-10)
    if alg == "incremental":
        assert rep["passes"] == 1 and rep["config"]["finalize"] is False


def test_seeded_runs_repeat_minus_timing(capsys, mat, monkeypatch):
    path, _ = mat
    for argv in (("run", "isma", path, "--k", "4", "--seed", "11"),
                 ("run", "isma", path, "--k", "4", "--seed", "11", "--rows", "--strategy", "ls"),
                 ("run", "incremental", path, "--k", "4", "--blocks", "3", "--seed", "11")):
        assert _strip(_run(capsys, *argv)) == _strip(_run(capsys, *argv))
    one = _run(capsys, "run", "isma", path, "--k", "4", "--seed", "11", "--threads", "1")
    four = _run(capsys, "run", "isma", path, "--k", "4", "--seed", "11", "--threads", "4")
    assert [t["remaining"] for t in one["traces"]] == [t["remaining"] for t in four["traces"]]
    assert four["config"]["threads"] == 4
    monkeypatch.setenv("PODSKETCH_SEED", "11")
    env = _run(capsys, "run", "isma", path, "--k", "4")
    assert env["config"]["seed"] == 11 and _strip(env)["sigma"] == _strip(one)["sigma"]
    monkeypatch.setenv("PODSKETCH_SEED", "eleven")
    assert cli.main(["run", "isma", path, "--k", "4"]) == 2


def test_reference_adds_angles_and_wedin(capsys, mat, tmp_path):
    path, a = mat
    rep = _run(capsys, "run", "isma", path, "--k", "3", "--seed", "2", "--tau", "0.999",
               "--reference", path)
    assert len(rep["angles"]["mode_degrees"]) == 3 and max(rep["angles"]["principal_degrees"]) < 1
    assert set(rep["wedin"]) >= {"r_norm", "s_norm", "omega_hat", "measure", "ceiling"}
    g = _run(capsys, "run", "gram", path, "--k", "3", "--reference", path)
    # the Gram path squares the conditioning: agreement to ~1e-7 rad
    assert max(g["angles"]["principal_degrees"]) < 1e-5 and "wedin" in g


def test_save_factor_and_compare(capsys, mat, tmp_path):
    path, a = mat
    fpath = str(tmp_path / "f.podf")
    rep = _run(capsys, "run", "isma", path, "--k", "3", "--seed", "5", "--save-factor", fpath)
    f = pod.read_factor(fpath)
    np.testing.assert_array_equal(f.sigma[:3], rep["sigma"])
    same = _run(capsys, "compare", fpath, fpath, "--k", "3")
    assert max(same["angles"]["principal_degrees"]) < 1e-5
    assert max(same["angles"]["mode_degrees"]) < 1e-5
    e1 = np.eye(6)[:, :2]
    e2 = np.eye(6)[:, 2:4]
    pod.write_factor(str(tmp_path / "x.podf"), pod.TruncatedFactor(e1, np.array([2.0, 1.0])))
    pod.write_factor(str(tmp_path / "y.podf"), pod.TruncatedFactor(e2, np.array([2.0, 1.0])))
    dis = _run(capsys, "compare", str(tmp_path / "x.podf"), str(tmp_path / "y.podf"), "--k", "2")
    np.testing.assert_allclose(dis["angles"]["principal_degrees"], [90.0, 90.0])
    assert cli.main(["compare", fpath, path, "--k", "2"]) == 3  # subject must be a factor


def test_report_files_written(capsys, mat, tmp_path):
    path, _ = mat
    out = str(tmp_path / "rep.json")
    assert cli.main(["run", "isma", path, "--k", "3", "--seed", "1", "--out", out,
                     "--plots"]) == 0
    rep = json.load(open(out))
    reporting.validate_report(rep)
    for suffix in ("_sigma.csv", "_traces.csv"):
        assert os.path.exists(str(tmp_path / "rep") + suffix)


def test_exit_codes(capsys, mat, tmp_path):
    path, _ = mat
    assert cli.main(["run", "isma", path, "--k", "0"]) == 2
    assert cli.main(["run", "isma", str(tmp_path / "none.podm"), "--k", "2"]) == 3
    bad = tmp_path / "bad.podm"
    bad.write_bytes(b"PODM\x01\x00\x00\x00" + b"\x05" + b"\x00" * 7)
    assert cli.main(["run", "isma", str(bad), "--k", "2"]) == 3
    z = str(tmp_path / "z.podm")
    pod.write_matrix(z, np.zeros((10, 6)))
    assert cli.main(["run", "isma", z, "--k", "2"]) == 4


def test_module_invocation_end_to_end(mat, tmp_path):
    path, _ = mat
    out = str(tmp_path / "m.json")
    res = subprocess.run([sys.executable, "-m", "paper_1905_05107_b200", "run", "isma", path,
                          "--k", "2", "--out", out], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr
    reporting.validate_report(json.load(open(out)))


# ---- the reference CLI's own reports (tests/golden/make_cli_golden.py) ------
def _cli_golden():
    with open(os.path.join(ROOT, "tests", "golden", "cli_reports.json")) as f:
        return json.load(f)["cases"]


def _close(x, y, rtol, atol):
    np.testing.assert_allclose(np.asarray(x, dtype=float), np.asarray(y, dtype=float),
                               rtol=rtol, atol=atol)


@pytest.mark.parametrize("name", sorted(_cli_golden()))
def test_report_matches_reference_cli(capsys, tmp_path, name):
    """The drop-in's `run` report equals the report the reference's command
    line printed for the same matrix and arguments (reference cli.py run
    command + reporting.build_report): config echo, pass count and per-round
    bookkeeping exactly; sigma, cosines, angles and the Wedin block to fp64
    tolerance."""
    from golden.make_cli_golden import case_matrix, strip_timing

    case = _cli_golden()[name]
    path = str(tmp_path / "d.podm")
    pod.write_matrix(path, case_matrix())
    argv = [path if x == "MATRIX" else x for x in case["argv"]]
    got = strip_timing(_run(capsys, "run", *argv))
    ref = case["report"]
    assert sorted(got) == sorted(ref)
    assert got["config"] == ref["config"]
    assert got["passes"] == ref["passes"]
    _close(got["sigma"], ref["sigma"], 1e-10, 0)
    assert len(got["traces"]) == len(ref["traces"])
    for tg, tr in zip(got["traces"], ref["traces"]):
        assert sorted(tg) == sorted(tr)
        for key in ("iteration", "remaining", "columns_sampled", "rows_sampled"):
            assert tg[key] == tr[key], (key, tg, tr)
        assert len(tg["cosines"]) == len(tr["cosines"])
        _close(tg["cosines"], tr["cosines"], 0, 1e-9)
    if "angles" in ref:
        for key in ref["angles"]:
            # degrees; arccos near 1 resolves angles only to ~sqrt(eps) rad
            # (1e-6 deg), so an exact-reference run (gram) reads 0 .. 1e-5
            _close(got["angles"][key], ref["angles"][key], 0, 2e-5)
    if "wedin" in ref:
        for key, val in ref["wedin"].items():
            if isinstance(val, float):
                _close(got["wedin"][key], val, 1e-8, 1e-10)
            else:
                assert got["wedin"][key] == val, key
