"""Summarise an ncu capture of one kernel (ychg_scan_kernel, ychg_finish_kernel, ...) into profiles/ (json + markdown)."""
import csv, io, json, os, subprocess, sys

rep = sys.argv[1]
out_prefix = sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
def f(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__sass_inst_executed_op_global_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
summ = {k: {"value": f(k), "unit": u.get(k, "")} for k in keys if k in d}
stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
          for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
stalls = {k: v for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if v and v > 0.01}
rd = f("dram__bytes_read.sum"); wr = f("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd_b = rd * scale.get(u.get("dram__bytes_read.sum"), 1) if rd is not None else None
wr_b = wr * scale.get(u.get("dram__bytes_write.sum"), 1) if wr is not None else None
res = {"kernel": (d.get("Kernel Name") or "?").split("(")[0], "report": os.path.basename(rep), "metrics": summ, "stalls_per_issue": stalls,
       "dram_bytes_per_launch": (rd_b + wr_b) if rd_b is not None and wr_b is not None else None,
       "note": "one ncu --set full replay of one launch (cold-cache, serialised): shares, not absolutes"}
with open(out_prefix + ".json", "w") as fh:
    json.dump(res, fh, indent=1)
with open(out_prefix + ".md", "w") as fh:
    fh.write(f"# ncu summary: {res['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
    for k, v in summ.items():
        fh.write(f"| {k} | {v['value']} | {v['unit']} |\n")
    fh.write("\n## warp stall reasons (per issued instruction)\n\n| reason | ratio |\n|---|---|\n")
    for k, v in stalls.items():
        fh.write(f"| {k} | {v:.3f} |\n")
    fh.write(f"\nDRAM bytes per launch (read+write): {res['dram_bytes_per_launch']}\n")
print(json.dumps(res, indent=1)[:3000])
