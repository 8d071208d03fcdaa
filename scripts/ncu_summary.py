"""Summarize ncu --set full captures of the DSG sweep kernels into
profiles/ncu_traffic.json (dram bytes per launch, the number bench.py's
roofline.traffic quotes) and a readable text table (development aid)."""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefront_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "smem_dynamic_bytes"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
]
ROLE = {  # (C, MODE) -> role key used by bench.py
    ("1", "0"): "sweep_recompute_A", ("2", "0"): "sweep_recompute_B",
    ("1", "1"): "sweep_store", ("2", "2"): "sweep_cached", ("1", "2"): "apply_cached",
}

out = {"source": [], "kernels": {}}
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "Kbyte/block": 1e3, "byte/block": 1, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    out["source"].append(rep)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        targs = name[name.index("<") + 1:name.index(">")].replace(" ", "").split(",")
        key = ROLE.get((targs[2], targs[3]), name)
        m = {}
        for met, short in METRICS:
            if met in hdr:
                i = hdr.index(met)
                try:
                    m[short] = float(r[i].replace(",", "")) * scale.get(units[i], 1)
                except ValueError:
                    pass
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]))
        m["stalls_per_issue"] = {k: round(v, 3) for v, k in sorted(stalls, reverse=True)[:7]}
        m["kernel"] = name.split("(")[0]
        m["dram_bytes_per_launch"] = m.get("dram_read", 0) + m.get("dram_write", 0)
        out["kernels"][key] = m
if out["kernels"].get("sweep_recompute_A") and "sweep_recompute" not in out["kernels"]:
    a, b = out["kernels"].get("sweep_recompute_A"), out["kernels"].get("sweep_recompute_B")
    if a and b:
        out["kernels"]["sweep_recompute"] = {
            "kernel": "sweep A + sweep B (recompute)", "note": "sum of the two launches",
            "dram_bytes_per_launch": (a["dram_bytes_per_launch"] + b["dram_bytes_per_launch"]) / 2}
print(json.dumps(out, indent=1))
