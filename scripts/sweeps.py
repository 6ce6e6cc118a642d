"""BASELINE configs 3 and 4 on one B200, each point one bench.py run (K=20-step
graph, W=5, the driver's settings): the resolution sweep at fixed content --
frame (exactly 4 hyperedges at every size >= 3^2) from 32^2 to 512^2, hbands(147)
(exactly 147) from 1000^2 to 21000^2 -- locating the GPU/CPU crossover of the
end-to-end call against the reference on the host cores; and the hyperedge-count
sweep at 21000^2 (147 -> 220.5M hyperedges).  Writes gpurun_out/<tag>_sweeps.jsonl
and gpurun_out/<tag>_sweeps.md (copied into profiles/)."""
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
runs = []
for s in (32, 64, 128, 256, 512):
    runs.append(("resolution", ["--size", str(s), "--pattern", "frame"]))
for s in (1000, 2000, 4000, 8000, 12000, 16000, 21000):
    runs.append(("resolution", ["--size", str(s), "--pattern", "hbands", "--bands", "147"]))
for pat, arg, cpu in (("hbands", ["--bands", "147"], True), ("hbands", ["--bands", "10500"], True),
                      ("checker", ["--cell", "64"], True), ("checker", ["--cell", "21"], True),
                      ("checker", ["--cell", "10"], True), ("checker", ["--cell", "7"], True),
                      ("random", ["--density", "0.5", "--seed", "1307"], False),
                      ("checker", ["--cell", "1"], False)):
    runs.append(("hyperedges", ["--size", "21000", "--pattern", pat, *arg] + ([] if cpu else ["--no-cpu-baseline"])))
rows = []
for axis, args in runs:
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "20", "--warmup", "5",
                          "--cpu-reps", "3", *args], capture_output=True, text=True, timeout=1200)
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
                      "gpix_s": d["value"], "frac": d["roofline"]["frac"], "isolated_us": d.get("isolated_us"),
                      "e2e_ms": (d.get("e2e") or {}).get("ms_per_step"),
                      "e2e_dropin_ms": (d.get("e2e_dropin") or {}).get("ms_per_step"),
                      "cpu_ms": (cpu.get("spread_ms") or {}).get("median"), "cpu_serial_ms": cpu.get("serial_ms"),
                      "hyperedges": d["totals"]["hyperedges"]}), flush=True)
os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
with open(os.path.join(root, "gpurun_out", f"{tag}_sweeps.jsonl"), "w") as f:
    for d in rows:
        f.write(json.dumps(d) + "\n")
with open(os.path.join(root, "gpurun_out", f"{tag}_sweeps.md"), "w") as f:
    f.write("# BASELINE configs 3-4 on one B200 (bench.py per point: K=20-step graph, W=5; full path: "
            "counts+flags+boundaries+hyperedges; parity of every point with a CPU column checked by bench.py)\n\n")
    f.write("| axis | workload | hyperedges | device us/step | Gpix/s | HBM frac | isolated us | e2e pinned ms | "
            "e2e drop-in (pageable) ms | CPU ref parallel ms (cores) | CPU ref serial ms | drop-in vs CPU parallel |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for d in rows:
        cpu = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        dr = d.get("e2e_dropin") or {}
        cms = (cpu.get("spread_ms") or {}).get("median")
        ratio = f"{cms / dr['ms_per_step']:.2f}x" if cms and dr.get("ms_per_step") else "-"
        f.write(f"| {d['axis']} | {d['config']['workload']} | {d['totals']['hyperedges']} | {d['ms_per_step'] * 1e3:.2f} | "
                f"{d['value']:.0f} | {d['roofline']['frac']:.3f} | {d.get('isolated_us')} | {e2e.get('ms_per_step')} | "
                f"{dr.get('ms_per_step')} | {cms} ({cpu.get('cores', '-')}) | {cpu.get('serial_ms', '-')} | {ratio} |\n")
