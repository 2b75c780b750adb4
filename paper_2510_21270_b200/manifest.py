"""Run manifests and report documents of the reference (manifest.hpp,
pbs_main.cpp `run`) on the device path.

    python -m paper_2510_21270_b200.manifest run --manifest run.json
    python -m paper_2510_21270_b200.manifest sweep --manifest run.json --tau-list 0.5,0.9 --out s.csv

A manifest names PBST input stacks (q, k, v), the PipelineConfig and where
the output tensor and the report go (manifest.hpp:17-39).  Keys, defaults and
error texts follow manifest_from_json / pipeline_from_json
(manifest.hpp:96-172).  The run loads the tensors straight into device memory
(bf16), runs Algorithm 1 once per head like the CLI (pbs_main.cpp:197-232),
adds the true-mass attention_coverage to each head's report, writes the
output PBST in the manifest's precision and the report document
{"aggregate": ..., "heads": [...]} with report_to_json's fixed fields
(manifest.hpp:174-186) and aggregate_reports' rules (pbs_main.cpp:124-144).

Precision: `f32` manifests run the device's f32 path (the reference's f32
arithmetic: permutations and masks bit-exact, outputs within 1e-4).  The device
has no f64 path, so an `f64` manifest (the reference default, pipeline.hpp:35)
is refused with E_CONFIG unless the caller opts into a lower device precision
(`--device-precision f32|bf16`, or run_manifest(device_precision=...)); the
output file keeps the manifest's dtype.  Other differences, by design: there is
no N^2 limit on the coverage (pbs_main.cpp:202-207 refuses N^2 > 2^26 on the
CPU).

`workload` manifests (manifest.hpp:26-39) are generated on the host by the
library's restatement of the reference generator (pbs_generate_workload_head,
workload.hpp:145-198, bit-identical tensors in the manifest's precision), then
uploaded and run like `inputs`; `--seed` overrides the workload seed as the
CLI does (pbs_main.cpp:56).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import dataclass

from . import _lib

_STRATEGIES = ("none", "key_permute", "query_permute", "both")
_PRECISIONS = ("f32", "f64")


def _config_error(msg):
    return _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_CONFIG: " + msg)


def _expect_keys(j: dict, allowed, where):
    for key in j:
        if key not in allowed:
            raise _config_error(f'unknown key "{key}" in {where}')


def _read(j: dict, key, kind, default):
    if key not in j:
        return default
    v = j[key]
    ok = (isinstance(v, bool) if kind is bool else
          isinstance(v, str) if kind is str else
          isinstance(v, (int, float)) and not isinstance(v, bool) if kind is float else
          isinstance(v, int) and not isinstance(v, bool) and v >= 0)
    if not ok:
        raise _config_error(f'bad value for "{key}"')
    return kind(v)


@dataclass
class RunManifest:
    """RunManifest (manifest.hpp:28-39), `inputs` form; pipeline defaults of
    PipelineConfig (pipeline.hpp:30-37) and ForcedPolicy (block_selection.hpp:163-166)."""

    q: str = ""
    k: str = ""
    v: str = ""
    workload: dict | None = None  # WorkloadSpec fields (workload_from_json), or None for `inputs`
    block_size: int = 128
    segment_size: int = 256
    tau: float = 0.9
    strategy: str = "key_permute"
    precision: str = "f64"
    force_first_block: bool = True
    force_diagonal_band: bool = True
    scale: float = 0.0
    attention: str = ""
    report: str = ""

    def config(self):
        from . import ops
        return ops.make_config(block_size=self.block_size, segment_size=self.segment_size, tau=self.tau,
                               strategy=self.strategy, forced_first_block=self.force_first_block,
                               forced_diagonal_band=self.force_diagonal_band, scale=self.scale)


_WORKLOAD_DEFAULTS = {"kind": "gaussian", "n": 1024, "d": 64, "heads": 1, "seed": 0, "line_count": 8,
                      "line_strength": 150.0, "scatter": "scattered"}


def workload_from_json(j: dict) -> dict:
    """workload_from_json (manifest.hpp:76-93) + WorkloadSpec::validate
    (workload.hpp:30-37), the reference's defaults and error texts."""
    if not isinstance(j, dict):
        raise _config_error('bad value for "workload"')
    _expect_keys(j, tuple(_WORKLOAD_DEFAULTS), "workload")
    w = dict(_WORKLOAD_DEFAULTS)
    for key in ("kind", "scatter"):
        w[key] = _read(j, key, str, w[key])
    for key in ("n", "d", "heads", "seed", "line_count"):
        w[key] = _read(j, key, int, w[key])
    w["line_strength"] = _read(j, "line_strength", float, w["line_strength"])
    if w["kind"] not in _lib.WORKLOAD_KINDS:
        raise _config_error(f"unknown workload kind '{w['kind']}'")
    if w["scatter"] not in _lib.LINE_SCATTER:
        raise _config_error(f"unknown scatter mode '{w['scatter']}'")
    if w["n"] == 0 or w["d"] == 0 or w["heads"] == 0:
        raise _config_error("workload dims must be >= 1")
    if w["kind"] in ("vertical_lines", "mixed"):
        if w["line_count"] > w["n"]:
            raise _config_error("line count exceeds sequence length")
        if w["line_strength"] <= 0:
            raise _config_error("line strength must be > 0")
    return w


def manifest_from_json(j: dict) -> RunManifest:
    """manifest_from_json (manifest.hpp:143-166)."""
    if not isinstance(j, dict):
        raise _config_error("manifest must be a JSON object")
    _expect_keys(j, ("workload", "inputs", "pipeline", "outputs"), "manifest")
    if ("workload" in j) == ("inputs" in j):
        raise _config_error('manifest needs exactly one of "workload" or "inputs"')
    if "workload" in j:
        m = RunManifest(workload=workload_from_json(j["workload"]))
    else:
        inp = j["inputs"]
        _expect_keys(inp, ("q", "k", "v"), "inputs")
        q, k, v = (_read(inp, x, str, "") for x in ("q", "k", "v"))
        if not q or not k or not v:
            raise _config_error("inputs need all of q, k, v paths")
        m = RunManifest(q, k, v)
    p = j.get("pipeline", {})
    _expect_keys(p, ("block_size", "segment_size", "tau", "strategy", "precision", "force_first_block",
                     "force_diagonal_band", "scale"), "pipeline")
    m.block_size = _read(p, "block_size", int, m.block_size)
    m.segment_size = _read(p, "segment_size", int, m.segment_size)
    m.tau = _read(p, "tau", float, m.tau)
    m.strategy = _read(p, "strategy", str, m.strategy)
    m.precision = _read(p, "precision", str, m.precision)
    m.force_first_block = _read(p, "force_first_block", bool, m.force_first_block)
    m.force_diagonal_band = _read(p, "force_diagonal_band", bool, m.force_diagonal_band)
    m.scale = _read(p, "scale", float, m.scale)
    if m.strategy not in _STRATEGIES:
        raise _config_error(f"unknown permutation strategy '{m.strategy}'")
    if m.precision not in _PRECISIONS:
        raise _config_error(f"unknown precision '{m.precision}' (expected f32 or f64)")
    o = j.get("outputs", {})
    _expect_keys(o, ("attention", "report"), "outputs")
    m.attention = _read(o, "attention", str, "")
    m.report = _read(o, "report", str, "")
    return m


def load_manifest(path) -> RunManifest:
    """load_manifest (manifest.hpp:168-177)."""
    try:
        f = open(path)
    except OSError:
        raise _lib.IoError(_lib.PBS_ERR_IO, f"E_IO: cannot open manifest '{path}'") from None
    with f:
        try:
            j = json.load(f)
        except json.JSONDecodeError as e:
            raise _config_error(f"manifest is not valid JSON: {e}") from None
    return manifest_from_json(j)


def report_to_json(r: dict, coverage: float) -> dict:
    """report_to_json (manifest.hpp:179-186): exactly these fields, microseconds."""
    return {"block_density": r["block_density"], "causal_density_baseline": r["causal_density_baseline"],
            "attention_coverage": coverage, "selected_blocks": int(r["selected_blocks"]),
            "total_admissible_blocks": int(r["total_admissible_blocks"]),
            "timings_us": {"estimate": r["estimate_us"], "permute": r["permute_us"], "select": r["select_us"],
                           "attention": r["attention_us"], "unpermute": r["unpermute_us"]}}


def aggregate_reports(heads: list) -> dict:
    """aggregate_reports (pbs_main.cpp:124-144): means of the densities and the
    coverage, sums of the counts and of the stage timings."""
    agg = json.loads(json.dumps(heads[0]))
    if len(heads) == 1:
        return agg
    for key in ("block_density", "causal_density_baseline", "attention_coverage"):
        agg[key] = sum(r[key] for r in heads) / len(heads)
    for key in ("selected_blocks", "total_admissible_blocks"):
        agg[key] = sum(r[key] for r in heads)
    for key in ("estimate", "permute", "select", "attention", "unpermute"):
        agg["timings_us"][key] = sum(r["timings_us"][key] for r in heads)
    return agg


def device_dtype(m: RunManifest, device_precision=None):
    """The device element type for a manifest: its own precision when the device
    has it (f32), else the caller's explicit choice; f64 alone is refused."""
    import torch

    choice = device_precision or m.precision
    if choice == "f32":
        return torch.float32
    if choice == "bf16":
        return torch.bfloat16
    raise _config_error("precision f64 is not supported by the B200 device path (pass --device-precision f32 or "
                        "bf16 to run an f64 manifest at lower precision)")


def workload_tensors(m: RunManifest, dtype):
    """generate_workload (workload.hpp:200-213) in the manifest's precision on
    the host, every head, then to the device as [heads, n, d] of `dtype`."""
    import numpy as np
    import torch

    from . import ops

    w = m.workload
    spec = ops.workload_spec(**w)
    host_prec = "f32" if m.precision == "f32" else "f64"
    heads = [ops.generate_workload_head(spec, h, m.block_size, m.segment_size, host_prec) for h in range(w["heads"])]
    dev = torch.device("cuda", torch.cuda.current_device())
    return tuple(torch.from_numpy(np.stack([hd[i] for hd in heads])).to(dev).to(dtype) for i in range(3))


def _load_inputs(m: RunManifest, resolve, dt):
    """load_inputs' `inputs` branch (pbs_main.cpp:83-97) straight to the device."""
    from . import ops

    infos = [ops.tensor_info(resolve(x)) for x in (m.q, m.k, m.v)]
    hc = [i["heads"] for i in infos]
    if hc[0] != hc[1] or hc[1] != hc[2]:
        raise _config_error(f"q/k/v head counts differ ({hc[0]}, {hc[1]}, {hc[2]})")
    if hc[0] == 0:
        raise _config_error("inputs hold no heads")
    # pbs_attention's checks (pipeline.hpp:111-116), before any tensor is loaded
    (qr, qc), (kr, kc), (vr, vc) = ((i["rows"], i["cols"]) for i in infos)
    if qr != kr:
        raise _config_error(f"pipeline expects self-attention: N == M, got {qr} vs {kr}")
    if qc != kc or kr != vr or vc != kc:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_SHAPE: pipeline inputs have inconsistent shapes")
    q, k, v = (ops.load_tensor(resolve(x), dtype=dt) for x in (m.q, m.k, m.v))
    from_stack = any(i["ndim"] == 3 for i in infos)
    q, k, v = (x if x.dim() == 3 else x.unsqueeze(0) for x in (q, k, v))
    return q, k, v, from_stack


def run_manifest(m: RunManifest, base_dir=".", device_precision=None) -> dict:
    """The CLI's `run` (pbs_main.cpp:197-232) on the GPU; returns the report document."""
    import torch

    from . import ops

    def resolve(p):
        return p if os.path.isabs(p) else os.path.join(base_dir, p)

    dt = device_dtype(m, device_precision)
    if m.workload is not None:
        q, k, v = workload_tensors(m, dt)
        from_stack = q.shape[0] > 1  # generate_workload's heads (pbs_main.cpp:74-80)
    else:
        q, k, v, from_stack = _load_inputs(m, resolve, dt)
    cfg = m.config()
    outs, reports = [], []
    for h in range(q.shape[0]):
        qh, kh, vh = q[h:h + 1], k[h:h + 1], v[h:h + 1]
        res = ops.pbs_attention(qh, kh, vh, cfg, report=True, return_perms=True)
        cov = ops.attention_coverage(qh, kh, res.mask, res.sigma, res.pi, m.block_size, m.scale)
        outs.append(res.output)
        reports.append(report_to_json(res.report, float(cov[0])))
    if m.attention:
        out = torch.cat(outs, 0)
        ops.save_tensor(resolve(m.attention), out if (from_stack or len(outs) > 1) else out[0],
                        file_dtype=m.precision)
    doc = {"aggregate": aggregate_reports(reports), "heads": reports}
    text = json.dumps(doc, indent=2) + "\n"
    if m.report:
        try:
            with open(resolve(m.report), "w") as f:
                f.write(text)
        except OSError:
            raise _lib.IoError(_lib.PBS_ERR_IO, f"E_IO: cannot open '{resolve(m.report)}' for writing") from None
    else:
        sys.stdout.write(text)
    return doc


def format_sweep_csv(rows) -> str:
    """format_sweep_csv (pbs_main.cpp:236-247)."""
    out = ["tau,S,strategy,density,coverage,max_err,mean_err,time_us\n"]
    for r in rows:
        out.append("%.6g,%d,%s,%.6f,%.6f,%.9g,%.9g,%.1f\n" % (r.tau, r.segment_size, r.strategy, r.density,
                                                             r.coverage, r.max_err, r.mean_err, r.time_us))
    return "".join(out)


def sweep_manifest(m: RunManifest, base_dir=".", taus=(), segments=(), strategies=(), out_path="",
                   device_precision=None) -> str:
    """The CLI's `sweep` (pbs_main.cpp:248-267): density_sweep of head 0 for every
    strategy (sorted, unique), defaults from the manifest's pipeline."""
    from . import ops

    def resolve(p):
        return p if os.path.isabs(p) else os.path.join(base_dir, p)

    dt = device_dtype(m, device_precision)
    if m.workload is not None:
        q, k, v = workload_tensors(m, dt)
    else:
        q, k, v = (ops.load_tensor(resolve(x), dtype=dt) for x in (m.q, m.k, m.v))
    q, k, v = (x[:1] if x.dim() == 3 else x.unsqueeze(0) for x in (q, k, v))
    taus = list(taus) or [m.tau]
    segments = list(segments) or [m.segment_size]
    rows = []
    for name in sorted(set(strategies or [m.strategy])):
        if name not in _STRATEGIES:
            raise _config_error(f"unknown permutation strategy '{name}'")
        cfg = m.config()
        cfg.strategy = _lib.STRATEGIES[name]
        rows += ops.density_sweep(q, k, v, cfg, taus, segments)
    text = format_sweep_csv(rows)
    if out_path:
        with open(out_path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return text


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2510_21270_b200.manifest")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="Run the pipeline per head and write reports")
    r.add_argument("--manifest", required=True)
    r.add_argument("--device-precision", choices=["f32", "bf16"], default=None,
                   help="device element type (default: the manifest's precision; f64 needs this)")
    r.add_argument("--seed", type=int, default=None, help="Workload seed override")
    sw = sub.add_parser("sweep", help="Density/coverage/error sweep as CSV")
    sw.add_argument("--manifest", required=True)
    sw.add_argument("--tau-list", default="")
    sw.add_argument("--segment-list", default="")
    sw.add_argument("--strategies", default="")
    sw.add_argument("--out", default="")
    sw.add_argument("--device-precision", choices=["f32", "bf16"], default=None)
    sw.add_argument("--seed", type=int, default=None, help="Workload seed override")
    args = ap.parse_args(argv)
    try:
        m = load_manifest(args.manifest)
        if args.seed is not None and m.workload is not None:  # apply_overrides (pbs_main.cpp:56)
            m.workload["seed"] = args.seed
        base = os.path.dirname(os.path.abspath(args.manifest))
        if args.cmd == "run":
            run_manifest(m, base, args.device_precision)
        else:
            split = lambda s: [x for x in s.split(",") if x]  # noqa: E731
            sweep_manifest(m, base, [float(x) for x in split(args.tau_list)],
                           [int(x) for x in split(args.segment_list)], split(args.strategies), args.out,
                           args.device_precision)
    except _lib.PbsError as e:  # the CLI's stderr line and exit code (pbs_main.cpp:467-480)
        sys.stderr.write(str(e) + "\n")
        return e.code
    return 0


if __name__ == "__main__":
    sys.exit(main())
