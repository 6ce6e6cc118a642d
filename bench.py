#!/usr/bin/env python3
"""yCHG hot-path benchmark (BASELINE.json metric: Gpixel/s and achieved HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--size 21000] [--pattern hbands] [--bands 147]

One "step" = one pass of the hot path over one synthetic mask: per-column
cut-vertex counts + change flags + ascending boundary list + hyperedge total
(== hyperedge_count(decompose(build_profile(img))) in the reference).

N=1 workload = BASELINE config[1]: a 21000x21000 mask with a fixed hyperedge
count (hbands(147) -> exactly 147 hyperedges), generated bit-exactly on the
device by K0.  N>1 (torchrun, one rank per GPU): weak scaling, each rank owns a
21000-column strip of a (21000*N)x21000 mask (+ an 8-column right halo), counts
are all-gathered and links all-reduced over NCCL.

Timing: W untimed warm-up steps; K timed steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.  The 55 MB
mask fits in the 126 MB L2, so consecutive steps rotate over >= 5 distinct
device copies (>= 275 MB between reuses).  `e2e` times the public host API
(ychg_scan_host: pinned H2D + kernels + D2H of counts/boundaries/totals).
"""
from __future__ import annotations

import argparse
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
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=21000, help="square mask side (per-rank strip width for N>1)")
    ap.add_argument("--height", type=int, default=0, help="override height (default = size)")
    ap.add_argument("--pattern", default="hbands", choices=["hbands", "random", "checker", "full", "frame"])
    ap.add_argument("--bands", type=int, default=147)
    ap.add_argument("--cell", type=int, default=7)
    ap.add_argument("--density", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=1307)
    ap.add_argument("--counts-only", action="store_true", help="skip K3 (hyperedge total)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--emulate-collectives", action="store_true",
                    help="N=1 only: run the N>1 side-stream/event structure with local copies (tests the graph)")
    ap.add_argument("--cpu-reps", type=int, default=3)
    return ap.parse_args()


HOLD_NOTE = ("spin kernel holds the stream while the host submits the timed work, so the region "
             "measures device execution, not graph-submission latency (nvbench's blocking-kernel method)")


def hold_cycles(steps: int) -> int:
    """Spin length before the start event: ~10 us of submission budget per step, >= 0.2 ms.
    YCHG_BENCH_HOLD_CYCLES overrides (0 disables)."""
    v = os.environ.get("YCHG_BENCH_HOLD_CYCLES")
    return int(v) if v is not None else max(400_000, 20_000 * steps)


def hold_stream(stream, steps: int) -> bool:
    """Enqueue the hold; False (no hold, the region then includes submission) if torch lacks _sleep."""
    n = hold_cycles(steps)
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
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def profiled_traffic(algorithmic_bytes):
    """dram bytes per launch of the scan kernel from the committed ncu capture (made
    on the default 21000^2 workload), if this run is that workload."""
    p = os.path.join(ROOT, "profiles", "ncu_scan_summary.json")
    try:
        with open(p) as f:
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
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_name(a, W, H):
    pat = {"hbands": f"hbands({a.bands})", "random": f"random({a.density},{a.seed})",
           "checker": f"checker({a.cell})", "full": "full", "frame": "frame"}[a.pattern]
    return f"{W}x{H} {pat} mask"


def expected_hyperedges(a, W, H):
    if a.pattern == "hbands":
        return a.bands
    if a.pattern == "full":
        return 1
    if a.pattern == "frame":
        return 4 if W >= 3 and H >= 3 else None
    return None


# ---------------------------------------------------------------------------- reference arm
def cpu_reference(a, W, H, reps, warmup, bits=None):
    """The unmodified reference CPU path (oracle/_ref) on the host cores: counts
    (parallel(nproc)) + boundaries + hyperedge_count(decompose(build_profile))."""
    from oracle import PATTERN_IDS, Reference, Spec

    ref = Reference()
    nproc = os.cpu_count() or 1
    if bits is not None:
        img = ref.image(bits, W)
    else:
        spec = Spec(PATTERN_IDS[a.pattern], W, H, a.bands if a.pattern == "hbands" else 0,
                    a.cell if a.pattern == "checker" else 0, a.density if a.pattern == "random" else 0.0,
                    a.seed if a.pattern == "random" else 0)
        img = ref.image_synth(spec)
    r = img.time_path(1, nproc, warmup, reps, with_hyperedges=not a.counts_only)
    ns = sorted(r["ns"])
    med = ns[(len(ns) - 1) // 2]  # lower median, bench.cpp:21-25
    return {"gpix_s": W * H / (med * 1e-9) / 1e9, "median_ms": med / 1e6, "ns": r["ns"], "cores": nproc,
            "hyperedges": r["hyperedges"], "n_boundaries": r["n_boundaries"]}


def run_reference_arm(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    W = a.size * max(1, a.gpus) if a.gpus > 1 else a.size
    H = a.height or a.size
    reps = max(1, min(a.steps, 5))
    t0 = time.time()
    r = cpu_reference(a, W, H, reps, min(a.warmup, 1))
    line = {
        "impl": "reference", "metric": "Gpixel/s", "value": round(r["gpix_s"], 4), "unit": "Gpixel/s",
        "n_gpus": a.gpus, "steps": reps, "warmup": min(a.warmup, 1), "ms_per_step": round(r["median_ms"], 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8 (1 bit/pixel), int32 counts",
        "data": "synthetic (reference synth)",
        "config": {"workload": workload_name(a, W, H), "width": W, "height": H,
                   "path": "counts" + ("" if a.counts_only else "+boundaries+hyperedge_count(decompose(build_profile))")},
        "cpu_baseline": {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "cores": r["cores"], "kind": "reference",
                         "sample": f"full {W}x{H} mask, lower median of {reps} reps, parallel({r['cores']})"},
        "e2e": {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "hyperedges": r["hyperedges"], "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def run_ours(a):
    import numpy as np
    import torch

    import paper_1307_2560_b200 as y

    world, rank, local = dist_env()
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE={world}"
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
    sptr = stream.cuda_stream

    H = a.height or a.size
    Ws = a.size                             # counted columns on this rank
    W_total = Ws * world
    halo = 8 if (world > 1 and rank < world - 1) else 0
    Wimg = Ws + halo
    pitch = y.pitch_for(Wimg)
    img_bytes = H * ((Ws + 7) // 8)         # algorithmic bytes of this rank's mask (unpadded)
    L2 = torch.cuda.get_device_properties(local).L2_cache_size
    nbuf = max(5, -(-4 * L2 // max(1, pitch * H)))
    nbuf = min(nbuf, 16)
    bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(nbuf)]
    kw = dict(bands=a.bands if a.pattern == "hbands" else 0, cell=a.cell if a.pattern == "checker" else 0,
              density=a.density if a.pattern == "random" else 0.0, seed=a.seed if a.pattern == "random" else 0)
    if a.pattern == "random" and world > 1:
        raise SystemExit("multi-GPU bench uses column-independent patterns (hbands/checker/full)")
    for b in bufs:
        y.synth_device(a.pattern, Wimg, H, b.data_ptr(), pitch, stream=sptr, **kw)
    # Per-step output slots (R of them, R > steps): the collectives of step i run on
    # a side stream while the next steps scan into other slots, so the streaming
    # pipeline (PDL between consecutive scans) never waits on a collective; a slot
    # is only reused after its collectives completed (event wait).
    R = a.steps + 1 if (dist is not None or a.emulate_collectives) else 2
    counts2 = [torch.empty(Ws, dtype=torch.int32, device="cuda") for _ in range(R)]
    flags = torch.empty((Ws + 31) // 32 + 32, dtype=torch.int32, device="cuda")
    bounds = torch.empty(Ws, dtype=torch.int32, device="cuda")
    totals2 = [torch.zeros(4, dtype=torch.int64, device="cuda") for _ in range(R)]
    collective = dist is not None or a.emulate_collectives
    gathered2 = [torch.empty(world * Ws, dtype=torch.int32, device="cuda") for _ in range(R)] if collective else None
    tsum2 = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(R)] if collective else None
    side = torch.cuda.Stream() if collective else None
    plan = y.Plan(Wimg, H, width_cnt=Ws, device=local)
    info = plan.info()
    with_links = not a.counts_only
    pending = [None] * R

    def step(i, s_main):
        """One step: the scan of input i on s_main; for N>1 the all-gather of the
        strip counts and the all-reduce of (runs, links) follow on the side stream,
        overlapped with the next steps' scans."""
        h = i % R
        if pending[h] is not None:
            s_main.wait_event(pending[h])  # an earlier step's collectives still read this slot
            pending[h] = None
        b = bufs[i % nbuf]
        plan.scan_device(b.data_ptr(), pitch, counts2[h].data_ptr(), flags.data_ptr(), bounds.data_ptr(),
                         totals2[h].data_ptr(), s_main.cuda_stream, with_links)
        if not collective:
            return
        ev = torch.cuda.Event()
        ev.record(s_main)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            if dist is not None:
                dist.all_gather_into_tensor(gathered2[h], counts2[h])
                tsum2[h].copy_(totals2[h][:2])
                dist.all_reduce(tsum2[h])
            else:  # --emulate-collectives (1 GPU): same stream/event structure, local copies
                gathered2[h][:Ws].copy_(counts2[h])
                tsum2[h].copy_(totals2[h][:2])
        done = torch.cuda.Event()
        done.record(side)
        pending[h] = done

    def join(s_main):
        if collective:
            s_main.wait_stream(side)
        for k in range(R):
            pending[k] = None

    for i in range(a.warmup):
        step(i, stream)
    join(stream)
    torch.cuda.synchronize()
    last = (a.warmup - 1) % R
    counts, totals = counts2[last], totals2[last]
    # sanity: the synthetic workload's known answer
    tot = totals.cpu().tolist()
    exp = expected_hyperedges(a, Ws, H)
    if world == 1 and with_links and exp is not None and tot[2] != exp:
        raise SystemExit(f"hyperedge total {tot[2]} != expected {exp}: refusing to report a number")
    if dist is not None:
        # the all-gathered counts are the global counts (column strips, rank order)
        g = gathered2[last]
        if not torch.equal(g[rank * Ws:(rank + 1) * Ws], counts):
            raise SystemExit("all-gathered counts do not match this rank's strip")

    # The K timed steps are one CUDA graph (two kernel nodes per step, plus the
    # collective nodes on a forked side stream for N>1), so the device runs them
    # back to back with no host launch overhead between steps.
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    try:
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap, capture_error_mode="thread_local"):
                cs = torch.cuda.current_stream()
                if collective:
                    side.wait_stream(cs)
                for i in range(a.steps):
                    step(a.warmup + i, cs)
                join(cs)
        stream.wait_stream(cap)
        graph.replay()  # warm replay
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001 -- e.g. a collective that refuses graph capture (N>1)
        if dist is None:
            raise
        print(f"[bench] CUDA-graph capture with collectives failed ({e!r}); timing eager steps", file=sys.stderr)
        graph = None
        for k in range(R):
            pending[k] = None
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    held = hold_stream(stream, a.steps)
    ev0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for i in range(a.steps):
            step(a.warmup + i, stream)
        join(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    if world == 1 and with_links and exp is not None and graph is not None:
        last_t = totals2[(a.warmup + a.steps - 1) % R] if R > 2 else totals2[(a.warmup + a.steps - 1) & 1]
        if int(last_t[2].item()) != exp:
            raise SystemExit("hyperedge total of the timed graph's last step != expected: refusing to report")
    # The north-star subset (K1 + K2: counts, change flags, boundaries, no K3
    # hyperedge total) timed the same way on the same inputs, reported beside the
    # headline (1 GPU only).
    alt = None
    if world == 1 and with_links:
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g2, stream=cap, capture_error_mode="thread_local"):
                cs2 = torch.cuda.current_stream().cuda_stream
                for i in range(a.steps):
                    b = bufs[(a.warmup + i) % nbuf]
                    plan.scan_device(b.data_ptr(), pitch, counts.data_ptr(), flags.data_ptr(), bounds.data_ptr(),
                                     totals.data_ptr(), cs2, False)
        stream.wait_stream(cap)
        g2.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hold_stream(stream, a.steps)
        e0.record(stream)
        g2.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / a.steps
        peak2, _ = measured_peak()
        alt = {"path": "counts+flags+boundaries (K1+K2, no K3 hyperedge total)",
               "value": round(W_total * H / (ms2 * 1e-3) / 1e9, 3), "unit": "Gpixel/s",
               "ms_per_step": round(ms2, 5), "roofline_frac": round(img_bytes / (ms2 * 1e-3) / 1e9 / peak2, 4)}
        del g2
    # eager leg (host-driven launches, one CUDA-event pair per scan) for reference
    plan.set_timing(True)
    eager_ms = []
    for i in range(min(a.steps, 10)):
        b = bufs[i % nbuf]
        plan.scan_device(b.data_ptr(), pitch, counts.data_ptr(), flags.data_ptr(), bounds.data_ptr(),
                         totals.data_ptr(), sptr, with_links)
        eager_ms.append(plan.last_ms()[0])
    plan.set_timing(False)
    clk = clocks.stop()
    if with_links and world == 1 and exp is not None and int(totals[2].item()) != exp:
        raise SystemExit("hyperedge total changed after graph replay")
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = t.item()
    # per-step average of the in-graph pipeline (stream kernel + its co-resident finisher)
    scan_avg = ms_total / a.steps
    ms_step = ms_total / a.steps
    pixels_all = W_total * H
    value = pixels_all / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    achieved = img_bytes / (scan_avg * 1e-3) / 1e9
    n_b = int(totals[3].item())

    e2e = None
    if not a.no_e2e and world == 1:
        host = torch.empty((H, (Ws + 7) // 8), dtype=torch.uint8, pin_memory=True)
        host.copy_(bufs[0][:, : (Ws + 7) // 8].cpu())
        himg = y.BinaryImage(Ws, H, host.numpy())
        for _ in range(2):
            y.scan(himg, with_hyperedges=with_links)
        ts = []
        for _ in range(max(3, min(a.steps, 30))):
            t0 = time.perf_counter()
            r = y.scan(himg, with_hyperedges=with_links)
            ts.append(time.perf_counter() - t0)
        if with_links and exp is not None and r.hyperedges != exp:
            raise SystemExit("e2e hyperedge total mismatch")
        t_med = sorted(ts)[len(ts) // 2]
        # the PCIe floor on this box: a bare pinned H2D copy of the same bytes (context only)
        dev = torch.empty_like(host, device="cuda")
        fl = []
        for _ in range(max(3, min(a.steps, 30))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.copy_(host, non_blocking=True)
            torch.cuda.synchronize()
            fl.append(time.perf_counter() - t0)
        del dev
        f_med = sorted(fl)[len(fl) // 2]
        # the same call on PAGEABLE rows (what the C++ drop-in receives from a reference
        # BinaryImage's std::vector): pinned staging pipeline inside ychg_scan_host
        pimg = y.BinaryImage(Ws, H, host.numpy().copy())
        y.scan(pimg, with_hyperedges=with_links)
        pts = []
        for _ in range(max(3, min(a.steps, 30))):
            t0 = time.perf_counter()
            y.scan(pimg, with_hyperedges=with_links)
            pts.append(time.perf_counter() - t0)
        p_med = sorted(pts)[len(pts) // 2]
        del pimg
        e2e = {"value": round(Ws * H / t_med / 1e9, 3), "unit": "Gpixel/s",
               "h2d_bytes_per_step": img_bytes, "d2h_bytes_per_step": 4 * Ws + 32 + 4 * n_b,
               "ms_per_step": round(t_med * 1e3, 3), "api": "ychg_scan_host (pinned host buffer)",
               "h2d_copy_floor_ms": round(f_med * 1e3, 3),
               "h2d_copy_gbs": round(host.numel() / f_med / 1e9, 2),
               "frac_of_copy_floor": round(f_med / t_med, 4),
               "pageable": {"value": round(Ws * H / p_med / 1e9, 3), "ms_per_step": round(p_med * 1e3, 3),
                            "note": "same call on pageable rows (reference BinaryImage storage)"}}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            hb = bufs[0][:, : (Ws + 7) // 8].cpu().numpy()
            r = cpu_reference(a, Ws, H, a.cpu_reps, 1, bits=hb)
            cpu = {"value": round(r["gpix_s"], 4), "unit": "Gpixel/s", "cores": r["cores"], "kind": "reference",
                   "sample": f"full {Ws}x{H} mask, reference counts(parallel({r['cores']}))+boundaries"
                             + ("" if a.counts_only else "+hyperedge_count(decompose(build_profile))")
                             + f", lower median of {a.cpu_reps} reps ({r['median_ms']:.1f} ms)",
                   "hyperedges": r["hyperedges"]}
            if with_links and r["hyperedges"] != int(totals[2].item()):
                raise SystemExit(f"reference hyperedges {r['hyperedges']} != ours {int(totals[2].item())}")
        except FileNotFoundError as e:
            cpu = {"unavailable": str(e)}

    totals_json = {"total_runs": int(totals[0].item()), "links": int(totals[1].item()),
                   "hyperedges": int(totals[2].item()), "n_boundaries": n_b}
    if dist is not None:  # global (runs, links) from the all-reduce of the last timed step
        g = tsum2[(a.warmup + a.steps - 1) % R].cpu().tolist()
        totals_json = {"total_runs": g[0], "links": g[1], "hyperedges": g[0] - g[1] if with_links else -1,
                       "n_boundaries_rank0_strip": n_b}
    if rank == 0:
        line = {
            "metric": "Gpixel/s", "value": round(value, 3), "unit": "Gpixel/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 (1 bit/pixel), int32 counts, int64 totals",
            "data": "synthetic (on-device K0 synth, bit-exact reference synth)",
            "config": {"workload": workload_name(a, W_total, H), "width": W_total, "height": H,
                       "strip_width_per_gpu": Ws, "path": "counts+flags+boundaries" + ("" if a.counts_only else "+hyperedges"),
                       "l2": f"rotating {nbuf} device copies ({nbuf * pitch * H / 1e6:.0f} MB > L2 {L2 / 1e6:.0f} MB)",
                       "parallelism": f"column strips x{world}" if world > 1 else "1 GPU",
                       "plan": {"grid": info.grid, "n_strips": info.n_strips, "seg_per_strip": info.seg_per_strip}},
            "hbm_gbs_step": round((img_bytes + 4 * Ws + 4 * n_b + 32) / (ms_step * 1e-3) / 1e9, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": profiled_traffic(img_bytes),
                         "frac_of_nominal_7700": round(achieved / 7700.0, 4),  # HGX B200 HBM3e nominal, context only
                         "kernel": "ychg_scan_kernel + ychg_finish_kernel (2 PDL launches per step)",
                         "kernel_ms": round(scan_avg, 5), "algorithmic_bytes": img_bytes,
                         "peak_source": peak_src,
                         "timing": ("CUDA events around a K-step CUDA graph replay" if graph is not None
                                    else "CUDA events around K eager steps (graph capture with collectives failed)")
                         + (f"; a {HOLD_NOTE}" if held else "")},
            "eager_launch_ms": round(sorted(eager_ms)[len(eager_ms) // 2], 5),
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "north_star_subset": alt,
            "gpu_launches": info.kernels_per_scan * a.steps,  # per timed graph (the subset graph: as many again)
            "totals": totals_json,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    if os.environ.get("YCHG_BENCH_WATCHDOG"):  # diagnostics: dump the Python stacks if a run stalls
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["YCHG_BENCH_WATCHDOG"]), exit=True)
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
