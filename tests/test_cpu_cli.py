"""CLI / file-format / report host logic (reference cli.py, podio.py,
reporting.py semantics) that needs no GPU: convert, PODF round trips and
errors, report schema, plot re-rendering, exit codes."""

import io
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import cli, podio, reporting

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _csv(path, rows):
    with open(path, "w") as f:
        f.write("# comment\n\n")
        for r in rows:
            f.write(",".join(repr(float(x)) for x in r) + "\n")


def test_convert_csv_to_column_major_podm(tmp_path, capsys):
    rows = np.arange(12.0).reshape(3, 4) + 0.5
    src = tmp_path / "m.csv"
    _csv(src, rows)
    assert cli.main(["convert", str(src)]) == 0
    m, n, nrm = capsys.readouterr().out.split()
    assert (int(m), int(n)) == (3, 4) and float(nrm) == float(np.linalg.norm(rows))
    raw = open(str(src) + ".podm", "rb").read()
    assert raw[:4] == b"PODM" and struct.unpack("<IQQ", raw[4:24]) == (1, 3, 4)
    np.testing.assert_array_equal(np.frombuffer(raw[24:], "<f8"), rows.ravel(order="F"))


def test_convert_center_and_podm_round_trip(tmp_path, capsys, rng):
    src = tmp_path / "c.csv"
    _csv(src, np.ones((4, 5)) * np.arange(1, 5)[:, None])
    out = tmp_path / "c.podm"
    assert cli.main(["convert", str(src), "--center", "--out", str(out)]) == 0
    assert np.abs(pod.read_matrix(str(out))).max() == 0.0
    a = rng.standard_normal((7, 3))
    p1 = tmp_path / "a.podm"
    pod.write_matrix(str(p1), a)
    assert cli.main(["convert", str(p1), "--out", str(tmp_path / "b.podm")]) == 0
    assert open(p1, "rb").read() == open(tmp_path / "b.podm", "rb").read()
    centred = pod.mean_center_rows(a)
    np.testing.assert_allclose(pod.mean_center_rows(centred), centred, atol=1e-15)


@pytest.mark.parametrize("content", ["1,2\n3\n", "1,x\n"])
def test_bad_csv_exits_three(tmp_path, capsys, content):
    src = tmp_path / "bad.csv"
    src.write_text(content)
    assert cli.main(["convert", str(src)]) == 3
    assert "line" in capsys.readouterr().err
    assert cli.main(["convert", str(tmp_path / "missing.csv")]) == 3


def test_factor_round_trip_and_format_errors(rng):
    u = np.linalg.qr(rng.standard_normal((9, 3)))[0]
    f = pod.TruncatedFactor(u, np.array([3.0, 2.0, 1.0]), np.linalg.qr(
        rng.standard_normal((5, 3)))[0])
    buf = io.BytesIO()
    pod.write_factor(buf, f)
    raw = buf.getvalue()
    g = pod.read_factor(io.BytesIO(raw))
    assert np.array_equal(g.u, f.u) and np.array_equal(g.sigma, f.sigma)
    assert np.array_equal(g.v, f.v)
    for cut in (10, 24 + 8 * 27 + 4, 24 + 8 * 27 + 8 + 8, len(raw) - 5):
        with pytest.raises(pod.FormatError):
            pod.read_factor(io.BytesIO(raw[:cut]))
    bad = bytearray(raw)
    bad[24 + 8 * 27 + 8 + 24] = 7  # V flag
    with pytest.raises(pod.FormatError, match="flag"):
        pod.read_factor(io.BytesIO(bytes(bad)))
    h = pod.TruncatedFactor(u, np.array([1.0, 2.0, 3.0]) * 0 + np.array([3.0, 2.0, 1.0]))
    buf = io.BytesIO()
    pod.write_factor(buf, h)
    assert pod.read_factor(io.BytesIO(buf.getvalue())).v is None
    # a PODM matrix is not a factor
    buf = io.BytesIO()
    pod.write_matrix(buf, u)
    with pytest.raises(pod.FormatError):
        pod.read_factor(io.BytesIO(buf.getvalue()))


def test_read_matrix_validation(tmp_path):
    p = tmp_path / "nan.podm"
    with open(p, "wb") as f:
        f.write(podio.Podm(1, 2).pack())
        f.write(np.array([1.0, np.nan]).tobytes())
    with pytest.raises(pod.FormatError, match="non-finite"):
        pod.read_matrix(str(p))
    with open(p, "wb") as f:
        f.write(podio._LAYOUT.pack(b"PODX", 1, 1, 1))
    with pytest.raises(pod.FormatError, match="magic"):
        pod.read_matrix(str(p))
    a = pod.read_matrix(io.BytesIO(podio._LAYOUT.pack(b"PODM", 1, 2, 1) + b"\0" * 16))
    assert a.shape == (2, 1) and not a.flags.writeable


def _report(**extra):
    rep = {"config": {"algorithm": "isma", "k": 2, "tau": 0.99, "input": "a.podm"},
           "sigma": [2.0, 1.0],
           "traces": [{"iteration": 0, "columns_sampled": 5, "rows_sampled": 0,
                       "remaining": 10, "cosines": [], "wall_time": 0.1},
                      {"iteration": 1, "columns_sampled": 4, "rows_sampled": 0,
                       "remaining": 6, "cosines": [0.999, 0.5], "wall_time": 0.05}],
           "timing": {"wall_s": 0.2, "cpu_s": 0.1}, "passes": 3}
    rep.update(extra)
    return rep


def test_report_schema_and_serialisation():
    rep = _report(angles={"mode_degrees": [0.1, 0.2], "principal_degrees": [0.05, 0.2]})
    text = reporting.dump_report(rep)
    assert text.endswith("\n") and json.loads(text) == rep
    assert list(json.loads(text)) == sorted(rep)
    import jsonschema

    for bad in (dict(rep, extra=1), dict(rep, passes=-1),
                dict(rep, traces=[dict(rep["traces"][0], cosines=[1.5])]),
                {k: v for k, v in rep.items() if k != "timing"}):
        with pytest.raises(jsonschema.ValidationError):
            reporting.validate_report(bad)

    class W:
        r_norm, s_norm, omega_hat, measure, ceiling, degenerate = 1.0, 2.0, 0.0, np.inf, 3.0, True
        advisory = "increase k"

    w = reporting.wedin_to_json(W())
    assert w["measure"] is None and w["degenerate"] is True
    reporting.validate_report(dict(rep, wedin=w))


def test_plot_rerenders_saved_report(tmp_path, capsys):
    path = tmp_path / "r.json"
    path.write_text(reporting.dump_report(_report(
        angles={"mode_degrees": [0.1], "principal_degrees": [0.05, 0.2]})))
    assert cli.main(["plot", str(path), "--out-dir", str(tmp_path / "o")]) == 0
    out = capsys.readouterr().out.split()
    names = sorted(os.path.basename(p) for p in out)
    assert {"r_sigma.csv", "r_traces.csv", "r_angles.csv"} <= set(names)
    lines = open(tmp_path / "o" / "r_traces.csv").read().splitlines()
    assert lines[0].startswith("iteration,") and lines[1].split(",")[4] == ""
    assert lines[2].split(",")[4] == "0.5"
    ang = open(tmp_path / "o" / "r_angles.csv").read().splitlines()
    assert ang[2] == "2,,0.2"


def test_plot_rejects_non_reports(tmp_path, capsys):
    p = tmp_path / "x.json"
    p.write_text(json.dumps({"hello": 1}))
    assert cli.main(["plot", str(p)]) == 3
    p.write_text("not json")
    assert cli.main(["plot", str(p)]) == 3


def test_argparse_errors_exit_two(tmp_path):
    with pytest.raises(SystemExit) as e:
        cli.main(["run", "isma", "x.podm", "--k", "2", "--strategy", "bogus"])
    assert e.value.code == 2


def test_garbage_environment_seed_exits_two(monkeypatch):
    monkeypatch.setenv("PODSKETCH_SEED", "abc")
    with pytest.raises(pod.ParameterError):
        cli._resolve_seed(None)
    monkeypatch.setenv("PODSKETCH_SEED", "17")
    assert cli._resolve_seed(None) == 17 and cli._resolve_seed(3) == 3


def test_module_invocation_convert(tmp_path):
    src = tmp_path / "m.csv"
    _csv(src, [[1.0, 2.0], [3.0, 4.0]])
    res = subprocess.run([sys.executable, "-m", "paper_1905_05107_b200", "convert", str(src)],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0 and res.stdout.split()[:2] == ["2", "2"]
