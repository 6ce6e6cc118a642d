"""BASELINE configs 3 and 4 on one B200: the resolution sweep (1000^2 -> 21000^2,
fixed content hbands(147)) and the hyperedge-count sweep at 21000^2 (147 ->
220.5M hyperedges), each through bench.py (device-resident K-step graph, e2e via
ychg_scan_host, and the reference CPU path on the host cores where it fits).
Writes gpurun_out/<tag>_sweeps.jsonl and a markdown table (copied into profiles/)."""
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
runs = []
for s in (1000, 2000, 4000, 8000, 12000, 16000, 21000):
    runs.append(("resolution", ["--size", str(s), "--pattern", "hbands", "--bands", "147"]))
for pat, arg, cpu in (("hbands", ["--bands", "147"], True), ("hbands", ["--bands", "10500"], True),
                      ("checker", ["--cell", "64"], True), ("checker", ["--cell", "21"], True),
                      ("checker", ["--cell", "10"], True), ("checker", ["--cell", "7"], True),
                      ("checker", ["--cell", "1"], False)):
    runs.append(("hyperedges", ["--size", "21000", "--pattern", pat, *arg] + ([] if cpu else ["--no-cpu-baseline"])))
rows = []
for axis, args in runs:
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "100", "--warmup", "10",
                          "--cpu-reps", "3", *args], capture_output=True, text=True, timeout=900)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else ""
    try:
        d = json.loads(line)
    except Exception:  # noqa: BLE001
        print(axis, args, "FAILED", out.stderr[-800:], flush=True)
        continue
    d["axis"] = axis
    rows.append(d)
    cpu = d.get("cpu_baseline") or {}
    print(json.dumps({"axis": axis, "workload": d["config"]["workload"], "us_per_step": round(d["ms_per_step"] * 1e3, 2),
                      "gpix_s": d["value"], "frac": d["roofline"]["frac"], "e2e_gpix_s": (d.get("e2e") or {}).get("value"),
                      "cpu_gpix_s": cpu.get("value"), "hyperedges": d["totals"]["hyperedges"]}), flush=True)
os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
with open(os.path.join(root, "gpurun_out", f"{tag}_sweeps.jsonl"), "w") as f:
    for d in rows:
        f.write(json.dumps(d) + "\n")
with open(os.path.join(root, "gpurun_out", f"{tag}_sweeps.md"), "w") as f:
    f.write("# BASELINE configs 3-4 on one B200 (bench.py per point, K=100-step graph; full path: counts+flags+boundaries+hyperedges)\n\n")
    f.write("| axis | workload | hyperedges | device us/step | Gpix/s | HBM frac | e2e Gpix/s (H2D incl.) | CPU ref Gpix/s (cores) | GPU/CPU e2e |\n")
    f.write("|---|---|---|---|---|---|---|---|---|\n")
    for d in rows:
        cpu = d.get("cpu_baseline") or {}
        e2e = (d.get("e2e") or {}).get("value")
        ratio = f"{e2e / cpu['value']:.0f}x" if e2e and cpu.get("value") else "-"
        f.write(f"| {d['axis']} | {d['config']['workload']} | {d['totals']['hyperedges']} | {d['ms_per_step'] * 1e3:.2f} | "
                f"{d['value']:.0f} | {d['roofline']['frac']:.3f} | {e2e} | {cpu.get('value', '-')} ({cpu.get('cores', '-')}) | {ratio} |\n")
