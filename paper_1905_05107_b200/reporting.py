"""JSON run reports (reporting.py:1-295 of the reference): the schema the CLI
validates against, the trace / Wedin converters, canonical serialisation and
the comma-separated tables.  Figures need matplotlib, which this image does
not ship; without it ``render_plots`` notes that on stderr and writes none
(the tables are still written)."""

from __future__ import annotations

import csv
import json
import math
import sys


def _num(minimum=None, nullable=False):
    out = {"type": ["number", "null"] if nullable else "number"}
    if minimum is not None:
        out["minimum"] = minimum
    return out


def _int(minimum=None, nullable=False):
    out = {"type": ["integer", "null"] if nullable else "integer"}
    if minimum is not None:
        out["minimum"] = minimum
    return out


def _strict(required, props):
    return {"type": "object", "required": list(required), "additionalProperties": False,
            "properties": props}


def _build_schema():
    """Report layout (reporting.py:20-118): {config, sigma, traces, angles?,
    wedin?, timing, passes}; the nested objects other than config are
    closed."""
    config = {
        "type": "object",
        "required": ["algorithm", "k"],
        "properties": {
            "algorithm": {"type": "string"},
            "k": _int(1),
            "r": _int(nullable=True),
            "epsilon": _num(),
            "delta": _num(),
            "tau": _num(),
            "strategy": {"type": ["string", "null"]},
            "rows": {"type": "boolean"},
            "criterion": {"type": ["string", "null"]},
            "seed": _int(nullable=True),
            "finalize": {"type": "boolean"},
            "blocks": _int(nullable=True),
            "threads": _int(),
            "c": _int(nullable=True),
            "w": _int(nullable=True),
            "input": {"type": "string"},
            "reference": {"type": ["string", "null"]},
        },
    }
    trace = _strict(
        ("iteration", "columns_sampled", "rows_sampled", "remaining", "cosines", "wall_time"),
        {
            "iteration": _int(0),
            "columns_sampled": _int(0),
            "rows_sampled": _int(0),
            "remaining": _int(0),
            "cosines": {"type": "array",
                        "items": {"type": "number", "minimum": -1, "maximum": 1}},
            "wall_time": _num(0),
        })
    numbers = {"type": "array", "items": {"type": "number"}}
    angles = _strict(("mode_degrees", "principal_degrees"),
                     {"mode_degrees": numbers, "principal_degrees": numbers})
    wedin = _strict(
        ("r_norm", "s_norm", "omega_hat", "measure", "ceiling", "degenerate"),
        {
            "r_norm": _num(0),
            "s_norm": _num(0),
            "omega_hat": _num(0),
            "measure": _num(0, nullable=True),
            "ceiling": _num(0),
            "degenerate": {"type": "boolean"},
            "advisory": {"type": ["string", "null"]},
        })
    timing = _strict(("wall_s", "cpu_s"),
                     {"wall_s": _num(0), "cpu_s": _num(0), "flops_estimate": _num(0)})
    return {
        "$schema": "https://json-schema.org/draft/2020-12/schema",
        **_strict(("config", "sigma", "traces", "timing", "passes"), {
            "config": config,
            "sigma": numbers,
            "traces": {"type": "array", "items": trace},
            "angles": angles,
            "wedin": wedin,
            "timing": timing,
            "passes": _int(0),
        }),
    }


REPORT_SCHEMA = _build_schema()


def validate_report(report):
    """reporting.py:121-123 -- raise jsonschema.ValidationError if malformed."""
    import jsonschema

    jsonschema.validate(report, REPORT_SCHEMA)


def traces_to_json(traces):
    """reporting.py:126-137"""
    return [{"iteration": int(t.iteration), "columns_sampled": int(t.columns_sampled),
             "rows_sampled": int(t.rows_sampled), "remaining": int(t.remaining),
             "cosines": [float(x) for x in t.cosines], "wall_time": float(t.wall_time)}
            for t in traces]


def wedin_to_json(rep):
    """reporting.py:140-149 -- an infinite measure (degenerate gap) is null."""
    measure = float(rep.measure)
    return {"r_norm": float(rep.r_norm), "s_norm": float(rep.s_norm),
            "omega_hat": float(rep.omega_hat),
            "measure": None if math.isinf(measure) else measure,
            "ceiling": float(rep.ceiling), "degenerate": bool(rep.degenerate),
            "advisory": rep.advisory}


def dump_report(report):
    """reporting.py:152-155 -- validated, sorted keys, indent 2, newline."""
    validate_report(report)
    return json.dumps(report, indent=2, sort_keys=True) + "\n"


def write_report(report, path):
    with open(path, "w", encoding="utf-8") as f:
        f.write(dump_report(report))


def _write_csv(path, header, rows):
    with open(path, "w", newline="", encoding="utf-8") as f:
        wr = csv.writer(f)
        wr.writerow(header)
        wr.writerows(rows)
    return path


def write_delimited(report, stem):
    """reporting.py:163-222 -- <stem>_sigma.csv always, _traces.csv when the
    run has traces, _angles.csv with a reference comparison; floats written
    with repr (round-trip precision).  Returns the paths."""
    paths = [_write_csv(f"{stem}_sigma.csv", ["mode", "sigma"],
                        [[i, repr(float(s))] for i, s in enumerate(report["sigma"], start=1)])]
    if report["traces"]:
        rows = []
        for t in report["traces"]:
            cos = t["cosines"]
            rows.append([t["iteration"], t["columns_sampled"], t["rows_sampled"],
                         t["remaining"], repr(min(cos)) if cos else "", repr(t["wall_time"])])
        paths.append(_write_csv(
            f"{stem}_traces.csv",
            ["iteration", "columns_sampled", "rows_sampled", "remaining", "min_cosine",
             "wall_time"], rows))
    if "angles" in report:
        md, pd = report["angles"]["mode_degrees"], report["angles"]["principal_degrees"]
        rows = [[i + 1, repr(md[i]) if i < len(md) else "", repr(pd[i]) if i < len(pd) else ""]
                for i in range(max(len(md), len(pd)))]
        paths.append(_write_csv(f"{stem}_angles.csv",
                                ["mode", "mode_angle_deg", "principal_angle_deg"], rows))
    return paths


def render_plots(report, stem):
    """reporting.py:225-295 -- figures (sigma decay, convergence, angles)."""
    try:
        import matplotlib
    except ImportError:
        print("note: figures need matplotlib, which is not installed; tables only",
              file=sys.stderr)
        return []
    matplotlib.use("Agg")
    import matplotlib.pyplot as plt

    paths = []
    sigma = report["sigma"]
    if sigma:
        fig, ax = plt.subplots(figsize=(5, 3.5))
        ax.semilogy(range(1, len(sigma) + 1), sigma, "o-", ms=4)
        ax.set(xlabel="mode", ylabel="sigma_i", title="singular value decay")
        fig.tight_layout()
        paths.append(f"{stem}_sigma.png")
        fig.savefig(paths[-1], dpi=150)
        plt.close(fig)
    traced = [t for t in report["traces"] if t["cosines"]]
    if traced:
        fig, ax = plt.subplots(figsize=(5, 3.5))
        ax.plot([t["iteration"] for t in traced], [min(t["cosines"]) for t in traced], "o-")
        if report["config"].get("tau") is not None:
            ax.axhline(report["config"]["tau"], color="k", ls="--", lw=0.8)
        ax.set(xlabel="iteration", ylabel="convergence cosine", ylim=(0, 1.05))
        fig.tight_layout()
        paths.append(f"{stem}_convergence.png")
        fig.savefig(paths[-1], dpi=150)
        plt.close(fig)
    if "angles" in report:
        md, pd = report["angles"]["mode_degrees"], report["angles"]["principal_degrees"]
        fig, ax = plt.subplots(figsize=(5, 3.5))
        ax.bar([i + 0.8 for i in range(len(md))], md, width=0.4, label="mode angle")
        ax.bar([i + 1.2 for i in range(len(pd))], pd, width=0.4, label="principal angle")
        ax.set(xlabel="mode", ylabel="degrees", title="error angles vs reference")
        ax.legend()
        fig.tight_layout()
        paths.append(f"{stem}_angles.png")
        fig.savefig(paths[-1], dpi=150)
        plt.close(fig)
    return paths
