#!/usr/bin/env python3
"""yCHG hot-path benchmark (BASELINE.json metric: Gpixel/s and achieved HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--size S] [--pattern hbands|random|checker|full|frame] [--bands 147]

One "step" = one pass of the hot path over one synthetic mask: per-column
cut-vertex counts + change flags + ascending boundary list + hyperedge total
(== hyperedge_count(decompose(build_profile(img))) in the reference).

* N=1 workload = BASELINE config[1]: a 21000x21000 mask with a fixed hyperedge
  count (hbands(147) -> exactly 147 hyperedges), generated bit-exactly on the
  device by K0.
* N>1 = BASELINE config[4]: ONE 65536x65536 mask cut into N column strips (strong
  scaling, multigpu.py), one rank per GPU over NCCL.  Each rank generates its
  strip (+ an 8-column right halo) in place with K0's global column offset; a
  step = the strip scan (counts and totals written straight into the all-gather
  segment) + ONE NCCL all-gather + two small kernels over the gathered buffer
  (global counts, the global boundary list with every strip's first-column
  fix-up, summed runs / links).  comm_ms / compute_ms are timed apart.
  Without WORLD_SIZE in the environment, `--gpus N` re-launches itself under
  torch.distributed.run with N ranks.

Timing: W untimed warm-up steps; K timed steps as one CUDA graph, bracketed by a
barrier + synchronize, CUDA events on the launching stream behind a spin kernel
(the host's graph submission is not timed), max over ranks.  Consecutive steps
rotate over distinct device copies of the mask (> 4x L2 between reuses).
`e2e` times the public API end to end from PINNED host rows (H2D + scan + D2H of
the results); `e2e_dropin` the same call on pageable rows (what the C++ drop-in
receives from a reference BinaryImage).  The reference CPU path is timed on the
same image (`cpu_baseline`) and its counts / boundaries / hyperedges are compared
with the last timed step (`parity`); a mismatch refuses to print a number.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=0, help="square mask side (default 21000 at N=1, 65536 at N>1)")
    ap.add_argument("--height", type=int, default=0, help="override height (default = size)")
    ap.add_argument("--pattern", default="hbands", choices=["hbands", "random", "checker", "full", "frame"])
    ap.add_argument("--bands", type=int, default=147)
    ap.add_argument("--cell", type=int, default=7)
    ap.add_argument("--density", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=1307)
    ap.add_argument("--counts-only", action="store_true", help="skip K3 (hyperedge total)")
    ap.add_argument("--no-skip", action="store_true", help="plan without the unchanged-block skip (A/B)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=3)
    a = ap.parse_args()
    if not a.size:
        a.size = 21000 if a.gpus == 1 else 65536
    return a


HOLD_NOTE = ("spin kernel holds the stream while the host submits the timed work, so the region "
             "measures device execution, not graph-submission latency (nvbench's blocking-kernel method)")


def hold_stream(stream, steps: int, per_step_cycles: int = 20_000) -> bool:
    """Spin before the start event: ~10 us of submission budget per step for one
    graph launch (>= 0.2 ms), ~100 us per step when the steps are submitted
    eagerly (collectives + kernels per step); YCHG_BENCH_HOLD_CYCLES overrides (0
    disables)."""
    v = os.environ.get("YCHG_BENCH_HOLD_CYCLES")
    n = int(v) if v is not None else max(400_000, per_step_cycles * steps)
    if n <= 0:
        return False
    import torch
    sleep = getattr(torch.cuda, "_sleep", None)
    if sleep is None:
        return False
    with torch.cuda.stream(stream):
        sleep(n)
    return True


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def profiled_traffic(algorithmic_bytes):
    """DRAM bytes per launch of the scan kernel from the committed ncu capture
    (profiles/ncu_scan_summary.json, made on the default 21000^2 workload), if
    this run is that workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_scan_summary.json")) as f:
            t = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None
    return t if t and abs(t - algorithmic_bytes) < 0.05 * algorithmic_bytes else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def relaunch_distributed(a) -> int:
    """`bench.py --gpus N` without a launcher: run N ranks under torch.distributed.run
    on this node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def workload_name(a, W, H):
    pat = {"hbands": f"hbands({a.bands})", "random": f"random({a.density},{a.seed})",
           "checker": f"checker({a.cell})", "full": "full", "frame": "frame"}[a.pattern]
    return f"{W}x{H} {pat} mask"


def synth_kwargs(a):
    return dict(bands=a.bands if a.pattern == "hbands" else 0, cell=a.cell if a.pattern == "checker" else 0,
                density=a.density if a.pattern == "random" else 0.0, seed=a.seed if a.pattern == "random" else 0)


def sha(arr) -> str:
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<i4").tobytes()).hexdigest()


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------- reference arm
def reference_image(a, W, H, bits=None):
    """A reference BinaryImage of the workload (reference synth, or given host rows)."""
    from oracle import PATTERN_IDS, Reference, Spec

    ref = Reference()
    if bits is not None:
        return ref, ref.image(bits, W)
    spec = Spec(PATTERN_IDS[a.pattern], W, H, a.bands if a.pattern == "hbands" else 0,
                a.cell if a.pattern == "checker" else 0, a.density if a.pattern == "random" else 0.0,
                a.seed if a.pattern == "random" else 0)
    return ref, ref.image_synth(spec)


def cpu_reference(a, W, H, reps, warmup, bits=None, serial=False):
    """The unmodified reference CPU path (oracle/_ref): counts (parallel(nproc)) +
    boundaries + hyperedge_count(decompose(build_profile)), timed with the
    reference protocol (bench.cpp:37-57: warm-up untimed, reps timed, lower median)."""
    import numpy as np

    ref, img = reference_image(a, W, H, bits)
    nproc = os.cpu_count() or 1
    r = img.time_path(1, nproc, warmup, reps, with_hyperedges=not a.counts_only)
    ns = sorted(r["ns"])
    med = ns[(len(ns) - 1) // 2]  # lower median, bench.cpp:21-25
    out = {"gpix_s": W * H / (med * 1e-9) / 1e9, "median_ms": med / 1e6, "min_ms": ns[0] / 1e6,
           "max_ms": ns[-1] / 1e6, "cores": nproc, "hyperedges": r["hyperedges"],
           "n_boundaries": r["n_boundaries"], "counts": np.asarray(r["counts"]).copy()}
    out["boundaries"] = ref.boundaries(out["counts"])
    if serial:  # one serial() rep, the reference's single-thread figure
        s = img.time_path(0, 1, 0, 1, with_hyperedges=not a.counts_only)
        out["serial_ms"] = s["ns"][0] / 1e6
    return out


def run_reference_arm(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    W = a.size
    H = a.height or a.size
    reps = max(1, min(a.steps, 5))
    t0 = time.time()
    r = cpu_reference(a, W, H, reps, min(a.warmup, 1))
    line = {
        "impl": "reference", "metric": "Gpixel/s", "value": round(r["gpix_s"], 4), "unit": "Gpixel/s",
        "n_gpus": a.gpus, "steps": reps, "warmup": min(a.warmup, 1), "ms_per_step": round(r["median_ms"], 3),
        "higher_is_better": True, "scaling": "strong" if a.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "u8 (1 bit/pixel), int32 counts", "data": "synthetic (reference synth)",
        "config": {"workload": workload_name(a, W, H), "width": W, "height": H,
                   "path": "counts" + ("" if a.counts_only else "+boundaries+hyperedge_count(decompose(build_profile))")},
        "cpu_baseline": {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "cores": r["cores"], "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"full {W}x{H} mask, lower median of {reps} reps, parallel({r['cores']})",
                         "spread_ms": {"min": round(r["min_ms"], 3), "median": round(r["median_ms"], 3),
                                       "max": round(r["max_ms"], 3)}},
        "e2e": {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "hyperedges": r["hyperedges"], "n_boundaries": r["n_boundaries"],
        "counts_sha256": sha(r["counts"]), "boundaries_sha256": sha(r["boundaries"]),
        "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def graph_time(torch, body, stream, steps, dist=None):
    """Capture `body(cs)` (K steps) as one CUDA graph and time one replay (ms), max
    over ranks; None if the capture fails (e.g. a collective that cannot be captured)."""
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    try:
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                body(torch.cuda.current_stream())
        stream.wait_stream(cap)
        g.replay()
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"[bench] CUDA-graph capture failed ({e!r}); timing eager steps", file=sys.stderr)
        torch.cuda.synchronize()
        g = None
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    held = hold_stream(stream, steps, 20_000 if g is not None else 200_000)
    e0.record(stream)
    if g is not None:
        g.replay()
    else:
        with torch.cuda.stream(stream):
            body(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    return ms, g is not None, held


def run_ours(a):
    import numpy as np
    import torch

    import paper_1307_2560_b200 as y
    from paper_1307_2560_b200.multigpu import StripExchange, plan_strips

    world, rank, local = dist_env()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}: launch with torchrun, or without a launcher")
    # YCHG_BENCH_SHARE_GPU=1 (function test of the N>1 code path on a 1-GPU box:
    # ranks share cuda:0 and talk over gloo; no number from such a run is valid)
    share = os.environ.get("YCHG_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    y._check(y._lib.ychg_set_device(local), "set_device")
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        if share:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    stream = torch.cuda.current_stream()
    with_links = not a.counts_only

    W = a.size
    H = a.height or a.size
    strips = plan_strips(W, world)
    s = strips[rank]
    Ws, Wimg = s.width_cnt, s.width_img
    pitch = y.pitch_for(Wimg)
    img_bytes = H * ((Ws + 7) // 8)          # algorithmic bytes of this rank's mask (unpadded)
    L2 = torch.cuda.get_device_properties(local).L2_cache_size
    nbuf = min(16, max(2, -(-4 * L2 // max(1, pitch * H)) + 1))
    bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(nbuf)]
    kw = synth_kwargs(a)
    for b in bufs:  # K0 with the strip's global column offset: bit-exact with the whole image's columns
        y.synth_device(a.pattern, W, H, b.data_ptr(), pitch, x0=s.c0, win=Wimg, stream=stream.cuda_stream, **kw)
    plan = y.Plan(Wimg, H, width_cnt=Ws, device=local, skip=not a.no_skip)
    info = plan.info()

    # Per-step outputs (R slots): the scan of step i writes slot i % R; for N>1 the
    # exchange of step i (one all-gather, then the assemble kernels) runs
    # on a side stream into the same slot while the next steps scan.
    R = a.steps + 1 if dist is not None else 2
    fw = y.boundary_flag_words(W)
    slots = []
    for _ in range(R):
        sl = {"counts": torch.empty(Ws, dtype=torch.int32, device="cuda"),
              "flags": torch.empty(fw, dtype=torch.int32, device="cuda"),
              "bounds": torch.empty(Ws, dtype=torch.int32, device="cuda"),
              "totals": torch.zeros(4, dtype=torch.int64, device="cuda")}
        if dist is not None:
            x = StripExchange(dist, strips, rank, device="cpu" if share else "cuda")
            sl["x"] = x
            if not share:  # the scan writes its counts and totals straight into the all-gather segment
                sl["counts"] = x.send[:Ws]
                sl["totals"] = x.totals_view
            sl["gcounts"] = torch.empty(W, dtype=torch.int32, device="cuda")
            sl["sums"] = torch.zeros(2, dtype=torch.int64, device="cuda")
            sl["gflags"] = torch.empty(fw, dtype=torch.int32, device="cuda")
            sl["gbounds"] = torch.empty(W, dtype=torch.int32, device="cuda")
            sl["gn"] = torch.zeros(1, dtype=torch.int64, device="cuda")
        slots.append(sl)
    side = torch.cuda.Stream() if dist is not None else None
    pending = [None] * R

    def scan(i, s_main, links=with_links, sl=None):
        sl = sl or slots[i % R]
        b = bufs[i % nbuf]
        plan.scan_device(b.data_ptr(), pitch, sl["counts"].data_ptr(), sl["flags"].data_ptr(),
                         sl["bounds"].data_ptr(), sl["totals"].data_ptr(), s_main.cuda_stream, links)

    def exchange(sl, s):
        """ONE NCCL all-gather of every strip's counts + totals, then two small kernels
        over the gathered buffer: the contiguous global counts, their change flags and
        boundary list (the strip-edge fix-up included), and the summed (runs, links)."""
        x = sl["x"]
        with torch.cuda.stream(s):
            if share:  # gloo: host tensors
                x.send[:Ws].copy_(sl["counts"].cpu())
                x.totals_view.copy_(sl["totals"].cpu())
                g = x.run().cuda()
            else:
                g = x.run()
            y.assemble_strips_device(g.data_ptr(), x.c0, x.seg, x.tot_off, sl["gcounts"].data_ptr(),
                                     sl["gflags"].data_ptr(), sl["gbounds"].data_ptr(), sl["gn"].data_ptr(),
                                     sl["sums"].data_ptr(), s.cuda_stream)

    def step(i, s_main):
        h = i % R
        if pending[h] is not None:
            s_main.wait_event(pending[h])  # an earlier step's exchange still reads this slot
            pending[h] = None
        scan(i, s_main)
        if dist is None:
            return
        ev = torch.cuda.Event()
        ev.record(s_main)
        side.wait_event(ev)
        exchange(slots[h], side)
        done = torch.cuda.Event()
        done.record(side)
        pending[h] = done

    def join(s_main):
        if side is not None:
            s_main.wait_stream(side)
        for k in range(R):
            pending[k] = None

    for i in range(a.warmup):
        step(i, stream)
    join(stream)
    torch.cuda.synchronize()

    def steps_body(cs):
        if side is not None:
            side.wait_stream(cs)
        for i in range(a.steps):
            step(a.warmup + i, cs)
        join(cs)

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms_total, graphed, held = graph_time(torch, steps_body, stream, a.steps, dist)
    last = slots[(a.warmup + a.steps - 1) % R]
    torch.cuda.synchronize()
    ms_step = ms_total / a.steps

    # N>1: compute alone (K strip scans) and the exchange alone (K exchanges of
    # finished counts), each timed the same way
    comm = None
    if dist is not None:
        ms_c, _, _ = graph_time(torch, lambda cs: [scan(a.warmup + i, cs, sl=slots[-1]) for i in range(a.steps)],
                                stream, a.steps, dist)
        ms_x, _, _ = graph_time(torch, lambda cs: [exchange(slots[(a.warmup + i) % R], cs) for i in range(a.steps)],
                                stream, a.steps, dist)
        comm = {"compute_ms": round(ms_c / a.steps, 5), "comm_ms": round(ms_x / a.steps, 5),
                "overlap": "each step's exchange runs on a side stream under the next steps' scans"}

    # N=1 extras: the K1+K2 subset, the no-skip A/B, one isolated scan
    alt = noskip = iso = None
    if dist is None and with_links:
        ms2, _, _ = graph_time(torch, lambda cs: [scan(a.warmup + i, cs, links=False, sl=slots[1])
                                                  for i in range(a.steps)], stream, a.steps)
        peak2, _ = measured_peak()
        alt = {"path": "counts+flags+boundaries (K1+K2, no K3 hyperedge total)",
               "value": round(W * H / (ms2 / a.steps * 1e-3) / 1e9, 3), "unit": "Gpixel/s",
               "ms_per_step": round(ms2 / a.steps, 5),
               "roofline_frac": round(img_bytes / (ms2 / a.steps * 1e-3) / 1e9 / peak2, 4)}
    if dist is None:
        other = y.Plan(Wimg, H, width_cnt=Ws, device=local, skip=a.no_skip)
        osl = slots[1]

        def body_ns(cs):
            for i in range(a.steps):
                b = bufs[(a.warmup + i) % nbuf]
                other.scan_device(b.data_ptr(), pitch, osl["counts"].data_ptr(), osl["flags"].data_ptr(),
                                  osl["bounds"].data_ptr(), osl["totals"].data_ptr(), cs.cuda_stream, with_links)
        ms3, _, _ = graph_time(torch, body_ns, stream, a.steps)
        noskip = {"skip": bool(a.no_skip), "ms_per_step": round(ms3 / a.steps, 5),
                  "value": round(W * H / (ms3 / a.steps * 1e-3) / 1e9, 3),
                  "note": "the same graph with the unchanged-block skip " + ("on" if a.no_skip else "off")}
        other.close()
        # one scan on an idle stream (CUDA events around the single launch), through a
        # latency plan (YCHG_PLAN_LATENCY: one CTA per SM, what an isolated caller uses)
        lp = y.Plan(Wimg, H, width_cnt=Ws, device=local, latency=True, skip=not a.no_skip)
        lp.set_timing(True)
        isl = []
        for i in range(25):
            b = bufs[i % nbuf]
            lp.scan_device(b.data_ptr(), pitch, osl["counts"].data_ptr(), osl["flags"].data_ptr(),
                           osl["bounds"].data_ptr(), osl["totals"].data_ptr(), stream.cuda_stream, with_links)
            isl.append(lp.last_ms()[0] * 1e3)
        # the same measurement of a near-empty kernel: the event/launch floor of any single launch
        fl = []
        for i in range(25):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.cuda._sleep(1)
            e1.record(stream)
            e1.synchronize()
            fl.append(e0.elapsed_time(e1) * 1e3)
        iso = {"us": round(sorted(isl[5:])[len(isl[5:]) // 2], 2), "plan": "YCHG_PLAN_LATENCY",
               "grid": lp.info().grid, "timing": "CUDA events around one launch on an idle stream, median of 20",
               "empty_kernel_us": round(sorted(fl[5:])[len(fl[5:]) // 2], 2)}
        lp.close()
    clk = clocks.stop()

    tot = last["totals"].cpu().tolist()
    value = W * H / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    achieved = img_bytes / (ms_step * 1e-3) / 1e9  # per-GPU HBM rate (each rank streams its strip)

    # ---- end to end through the public API, inputs from host memory every step
    e2e = e2e_dropin = None
    host = torch.empty((H, (Wimg + 7) // 8), dtype=torch.uint8, pin_memory=True)
    host.copy_(bufs[0][:, : (Wimg + 7) // 8].cpu())
    if not a.no_e2e and dist is None:
        himg = y.BinaryImage(Ws, H, host.numpy())
        for _ in range(2):
            y.scan(himg, with_hyperedges=with_links)
        ts = []
        for _ in range(max(5, min(a.steps, 30))):
            t0 = time.perf_counter()
            r = y.scan(himg, with_hyperedges=with_links)
            ts.append(time.perf_counter() - t0)
        if with_links and r.hyperedges != tot[2]:
            raise SystemExit("e2e hyperedge total differs from the device-resident scan: refusing to report")
        t_med = sorted(ts)[len(ts) // 2]
        dev = torch.empty_like(host, device="cuda")
        fl = []
        for _ in range(max(5, min(a.steps, 30))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.copy_(host, non_blocking=True)
            torch.cuda.synchronize()
            fl.append(time.perf_counter() - t0)
        del dev
        f_med = sorted(fl)[len(fl) // 2]
        e2e = {"value": round(Ws * H / t_med / 1e9, 3), "unit": "Gpixel/s",
               "h2d_bytes_per_step": img_bytes, "d2h_bytes_per_step": 4 * Ws + 32 + 4 * int(tot[3]),
               "ms_per_step": round(t_med * 1e3, 3), "api": "ychg_scan_host (pinned host rows)",
               "h2d_copy_floor_ms": round(f_med * 1e3, 3), "h2d_copy_gbs": round(host.numel() / f_med / 1e9, 2),
               "frac_of_copy_floor": round(f_med / t_med, 4)}
        # the drop-in's real input: a reference BinaryImage keeps its rows in a pageable std::vector
        pimg = y.BinaryImage(Ws, H, host.numpy().copy())
        y.scan(pimg, with_hyperedges=with_links)
        pts = []
        for _ in range(max(5, min(a.steps, 30))):
            t0 = time.perf_counter()
            y.scan(pimg, with_hyperedges=with_links)
            pts.append(time.perf_counter() - t0)
        p_med = sorted(pts)[len(pts) // 2]
        e2e_dropin = {"value": round(Ws * H / p_med / 1e9, 3), "unit": "Gpixel/s", "ms_per_step": round(p_med * 1e3, 3),
                      "api": "ychg::scan / ychg_scan_host on PAGEABLE rows (reference BinaryImage storage, image.hpp:71)",
                      "h2d_bytes_per_step": img_bytes}
        del pimg
    elif not a.no_e2e:
        # N>1: every step each rank copies its strip rows from pinned host memory,
        # scans, exchanges, and reads back the global boundary count + totals
        dimg = bufs[0]
        outs = torch.zeros(3, dtype=torch.int64, pin_memory=True)

        def e2e_body(cs):
            for i in range(a.steps):
                sl = slots[(a.warmup + i) % R]
                with torch.cuda.stream(cs):
                    dimg[:, : host.shape[1]].copy_(host, non_blocking=True)
                scan(0, cs, sl=sl)
                exchange(sl, cs)
                with torch.cuda.stream(cs):
                    outs[:2].copy_(sl["sums"], non_blocking=True)
                    outs[2:].copy_(sl["gn"], non_blocking=True)
        ms_e, _, _ = graph_time(torch, e2e_body, stream, a.steps, dist)
        e2e = {"value": round(W * H / (ms_e / a.steps * 1e-3) / 1e9, 3), "unit": "Gpixel/s",
               "h2d_bytes_per_step": img_bytes * world, "d2h_bytes_per_step": 24 * world,
               "ms_per_step": round(ms_e / a.steps, 5),
               "api": "per rank: pinned strip rows -> device (copy engine), ychg_scan_device, StripExchange "
                      "(NCCL), K2; D2H of (runs, links, n_boundaries); CUDA events, max over ranks"}

    # ---- parity of the last timed step and the reference CPU path on the same image
    cpu = parity = None
    if rank == 0 and not a.no_cpu_baseline:
        if dist is None:
            hb = host.numpy()[:, : (W + 7) // 8]
        else:  # the whole image, generated by K0 on this GPU (bit-exact with every strip)
            fpitch = y.pitch_for(W)
            full = torch.empty((H, fpitch), dtype=torch.uint8, device="cuda")
            y.synth_device(a.pattern, W, H, full.data_ptr(), fpitch, **kw)
            hb = full[:, : (W + 7) // 8].cpu().numpy()
            del full
        try:
            r = cpu_reference(a, W, H, a.cpu_reps if dist is None else 1, 1 if dist is None else 0, bits=hb,
                              serial=dist is None)
        except FileNotFoundError as e:
            r = None
            cpu = {"unavailable": str(e)}
        if r is not None:
            if dist is None:
                got_c = last["counts"].cpu().numpy()
                got_b = last["bounds"].cpu().numpy()[: int(tot[3])]
                got_he, got_nb = int(tot[2]), int(tot[3])
            else:
                got_c = last["gcounts"].cpu().numpy()
                got_nb = int(last["gn"].item())
                got_b = last["gbounds"].cpu().numpy()[:got_nb]
                sums = last["sums"].cpu().tolist()
                got_he = int(sums[0] - sums[1])
            parity = {"against": "reference counts(parallel) + detect_boundary_columns + "
                                 "hyperedge_count(decompose(build_profile)) on the same image (oracle/_ref)",
                      "step": "last timed step",
                      "counts_sha256_match": sha(got_c) == sha(r["counts"]),
                      "boundaries_match": bool(np.array_equal(got_b, r["boundaries"])),
                      "hyperedges_match": (not with_links) or got_he == r["hyperedges"],
                      "counts_sha256": sha(got_c), "boundaries_sha256": sha(got_b),
                      "n_boundaries": got_nb, "hyperedges": got_he if with_links else None}
            if not (parity["counts_sha256_match"] and parity["boundaries_match"] and parity["hyperedges_match"]):
                raise SystemExit(f"parity FAILED against the reference: {parity}: refusing to report a number")
            if dist is None:
                cpu = {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "cores": r["cores"], "kind": "reference",
                       "cpu_model": cpu_model(),
                       "sample": f"full {W}x{H} mask, reference counts(parallel({r['cores']}))+boundaries"
                                 + ("" if a.counts_only else "+hyperedge_count(decompose(build_profile))")
                                 + f", lower median of {a.cpu_reps} reps",
                       "spread_ms": {"min": round(r["min_ms"], 3), "median": round(r["median_ms"], 3),
                                     "max": round(r["max_ms"], 3)},
                       "serial_ms": round(r["serial_ms"], 3),
                       "serial_gpix_s": round(W * H / (r["serial_ms"] * 1e-3) / 1e9, 4),
                       "hyperedges": r["hyperedges"]}

    if rank == 0:
        totals_json = {"total_runs": int(tot[0]), "links": int(tot[1]), "hyperedges": int(tot[2]),
                       "n_boundaries": int(tot[3])}
        if dist is not None:
            sm = last["sums"].cpu().tolist()
            totals_json = {"total_runs": int(sm[0]), "links": int(sm[1]),
                           "hyperedges": int(sm[0] - sm[1]) if with_links else -1,
                           "n_boundaries": int(last["gn"].item())}
        line = {
            "metric": "Gpixel/s", "value": round(value, 3), "unit": "Gpixel/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "u8 (1 bit/pixel), int32 counts, int64 totals",
            "data": "synthetic (on-device K0 synth, bit-exact reference synth)",
            "config": {"workload": workload_name(a, W, H), "width": W, "height": H,
                       "strip_width_per_gpu": Ws, "halo_cols": s.halo_cols,
                       "path": "counts+flags+boundaries" + ("" if a.counts_only else "+hyperedges"),
                       "l2": f"rotating {nbuf} device copies per GPU ({nbuf * pitch * H / 1e6:.0f} MB > L2 {L2 / 1e6:.0f} MB)",
                       "parallelism": (f"{world} column strips, one {'gloo (shared-GPU function test)' if share else 'NCCL'} "
                                       "all-gather per step") if world > 1 else "1 GPU",
                       "plan": {"grid": info.grid, "n_strips": info.n_strips, "seg_per_strip": info.seg_per_strip,
                                "skip_unchanged_blocks": not a.no_skip}},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": profiled_traffic(img_bytes),
                         "kernel": "ychg_scan_kernel (one launch per step: stream + strip finish fused)",
                         "kernel_ms": round(ms_step, 5), "algorithmic_bytes": img_bytes,
                         "algorithmic_bytes_note": "H*ceil(W/8) mask bytes per GPU per step (+4W counts, "
                                                   "+4 per boundary: <0.2%)",
                         "peak_source": peak_src,
                         "timing": ("CUDA events around a K-step CUDA graph replay" if graphed
                                    else "CUDA events around K eager steps") + (f"; a {HOLD_NOTE}" if held else "")},
            "isolated_us": iso["us"] if iso else None, "isolated": iso, "north_star_subset": alt, "skip_ab": noskip, "multi_gpu": comm,
            "e2e": e2e, "e2e_dropin": e2e_dropin, "cpu_baseline": cpu, "parity": parity, "clocks": clk,
            "gpu_launches": info.kernels_per_scan * a.steps + (3 * a.steps if world > 1 else 0),  # + NCCL, assemble x2
            "totals": totals_json,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    if os.environ.get("YCHG_BENCH_WATCHDOG"):  # diagnostics: dump the Python stacks if a run stalls
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["YCHG_BENCH_WATCHDOG"]), exit=True)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(a))
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
