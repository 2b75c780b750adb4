"""Summarise one `ncu --set full` capture (a .ncu-rep) into the counters the
roofline claims rest on, and (with --traffic) write profiles/attn_traffic.json,
which bench.py reads for roofline.traffic (DRAM bytes per launch).

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep [--traffic WORKLOAD] > profiles/rNN_ncu_<kernel>.txt

--traffic WORKLOAD records the capture under the bench's config.workload key
(e.g. llama31_8b_attn_128k_pbs); bench.py reports roofline.traffic only for
the workload a capture was taken on, else null.
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.per_cycle_active",
    "smsp__inst_executed.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def main(path, traffic=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = dict(zip(head, r))
        unit = dict(zip(head, units))
        print(f"kernel: {rec.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in rec:
                print(f"  {k:<95} {rec[k]:>18} {unit[k]}")
        stalls = sorted(((float(rec[k].replace(',', '')), k[len(STALL):].replace('_per_issue_active.ratio', ''))
                         for k in head if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")), reverse=True)
        print("  stall reasons (warps per issue-active cycle):")
        for v, k in stalls[:10]:
            print(f"    {k:<30} {v:8.3f}")
        if traffic:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(rec["dram__bytes_read.sum"].replace(',', '')) * scale[unit["dram__bytes_read.sum"]]
            wr = float(rec["dram__bytes_write.sum"].replace(',', '')) * scale[unit["dram__bytes_write.sum"]]
            dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "attn_traffic.json")
            doc = json.load(open(dst)) if os.path.exists(dst) else {}
            if "dram_bytes_per_launch" in doc:  # the round-1 single-capture form
                doc = {}
            doc[traffic] = {"kernel": rec.get("Kernel Name", "")[:60], "dram_bytes_per_launch": rd + wr,
                            "dram_read": rd, "dram_write": wr, "source": os.path.basename(path),
                            "note": "ncu --set full --clock-control none, one attention launch of the bench step"}
            json.dump(doc, open(dst, "w"), indent=1)

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None)
