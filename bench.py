#!/usr/bin/env python3
"""bench.py -- B200 block-iterative PLE over F2 (BASELINE.json metric).

metric: "PLE wall time & effective HBM GB/s, 65536^2 random F2 matrix, 1-8 GPU"

A step = one complete PLE (gf2::block_iterative_ple semantics) of the
65536 x 65536 matrix from the F2-nonlinear counter generator (SURVEY.md 8(d),
seed 1, rank 65534), i.e. one pass of the hot path over one synthetic input.

value      = effective GB/s = algorithmic trailing-update bytes / device time,
             summed over all ranks' steps ("alg bytes" = sum over 64-column
             panel steps of 16*(m-r-rb)*(W-w-1)); every step
             restores the input from a pristine HBM copy inside the timed
             region (the 512 MiB D2D copy is counted in the time).
e2e        = the same metric through the C ABI drop-in gf2cu_ple() on pinned
             HOST buffers: H2D of the input + PLE + D2H of L\\E every step
             (the library uploads in row blocks and starts on the first one,
             and streams finished rows back while the kernel runs; the same
             call on pageable memory is reported beside it).
roofline   = trailing_update (the dominant kernel): algorithmic bytes per
             launch / average CUDA-event launch duration, vs the measured HBM
             copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline = the reference itself (oracle/_ref/libgf2ref.so, compiled from
             /root/reference headers with its Release flags), single-threaded,
             on a bounded sample (the leading 65536 x 8192 column block of the
             same matrix), rank 0 at N=1 only.

--impl reference runs that reference arm alone (rank 0; other ranks exit 0).
Multi-GPU (torchrun, N>1): the device-driven row-sharded PLE (peer.py,
csrc/ple_peer.cuh) on BASELINE config 5's 131072^2 at every N (strong
scaling); value = the matrix's algorithmic bytes / the max-over-ranks device
time. --host-sharded: the NCCL host-orchestrated path;
--replicas: independent single-GPU instances.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PLE wall time & effective HBM GB/s, 65536² random F2 matrix, 1–8 GPU"
UNIT = "GB/s"
N_DEFAULT = 65536
SEED = 1
REF_SAMPLE_COLS = 8192


def alg_bytes_from_history(m, n, rhist, rbhist):
    W = (n + 63) // 64
    tot = 0
    for w, (r, rb) in enumerate(zip(rhist, rbhist)):
        if r >= m or w + 1 >= W:
            continue
        tot += 16 * (m - r - rb) * (W - w - 1)
    return tot


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_capture(driver: int = 2):
    """The dominant kernel's committed ncu --set full capture summary
    (profiles/super_traffic.json or persistent_traffic.json)."""
    name = "super_traffic.json" if driver == 2 else "persistent_traffic.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return {}


def load_traffic(driver: int = 2):
    """DRAM bytes per algorithmic (K = 64) byte of the dominant kernel."""
    d = load_capture(driver)
    return d.get("dram_bytes_per_k64_alg_byte", d.get("dram_bytes_per_alg_byte"))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.
    nvidia-smi can take a second to start on a fresh box, so it is started
    (and its first sample awaited) before the timed region; begin()/stop()
    bracket the region and only the samples taken inside it are kept."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []  # (monotonic time, line)
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.monotonic() + 10.0
            while not self.lines and time.monotonic() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def begin(self):
        self.t0 = time.monotonic()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def stop(self):
        self.t1 = time.monotonic()
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)  # the sample that covers the region's end
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [ln for (ts, ln) in self.lines if t0 <= ts <= self.t1 + 0.03]
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in inside:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms),
                "window_s": round(self.t1 - t0, 3)}


def make_host_ctr(m, n, seed):
    """The ctr input on the host from the TEST-ONLY generator in oracle/
    (liboracle.so), so the CPU legs map no library of the product."""
    import oracle as O
    return O.fill_ctr(m, n, seed)


def ref_alg_bytes(m, cols, q):
    """SURVEY.md 8(d)'s algorithmic bytes (K = 64 panels) of a PLE with pivot
    columns q -- the same definition the device arm reports."""
    q = np.asarray(q, dtype=np.int64)
    rh, rbh, r = [], [], 0
    for w in range((cols + 63) // 64):
        rb = int(np.count_nonzero((q >= 64 * w) & (q < 64 * w + 64)))
        rh.append(r)
        rbh.append(rb)
        r += rb
    return alg_bytes_from_history(m, cols, rh, rbh)


# ------------------------------------------------------------------ CPU legs
def run_reference_sample(m, cols, seed, reps=1):
    """The compiled reference on the leading m x cols block of the ctr matrix."""
    import oracle as O
    Wc = (cols + 63) // 64
    # the ctr generator is keyed on the full row width: generate full rows, slice
    big = make_host_ctr(m, N_DEFAULT, seed)
    base = np.ascontiguousarray(big[:, :Wc])
    del big
    secs, last = [], None
    for _ in range(reps):
        a = base.copy()
        out, s = O.ref_ple(a, m, cols)
        secs.append(s)
        last = out
    return secs, ref_alg_bytes(m, cols, last.q), last.rank


def run_reference_full(n, seed):
    """The compiled reference on the whole n x n ctr matrix (BASELINE config
    5 at 65536^2: the GPU arm's exact workload). One run, ~4.5 min."""
    import oracle as O
    a = make_host_ctr(n, n, seed)
    out, secs = O.ref_ple(a, n, n)
    return secs, ref_alg_bytes(n, n, out.q), out.rank


def reference_arm(args, rank):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref/libgf2ref.so = gf2::block_iterative_ple compiled from the
    reference headers with its Release flags; it is single-threaded, so 1
    core). W warm-up + K timed steps on the bounded sample, then ONE run of
    the full 65536^2 config, which is the line's `value` (same config as the
    device arm); the sample's figure is kept in cpu_baseline."""
    if rank != 0:
        return
    m, cols = N_DEFAULT, REF_SAMPLE_COLS
    try:
        import oracle as O
        O.ref()
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}))
        return
    for _ in range(args.warmup):
        run_reference_sample(m, cols, SEED)
    t0 = time.perf_counter()
    secs_all, bytes_all = [], 0
    for _ in range(args.steps):
        secs, b, rk = run_reference_sample(m, cols, SEED)
        secs_all += secs
        bytes_all += b
    tsum = sum(secs_all)
    sample_val = bytes_all / tsum / 1e9
    full = None
    if not args.ref_sample_only:
        fsecs, fbytes, frk = run_reference_full(N_DEFAULT, SEED)
        full = {"seconds": round(fsecs, 3), "alg_bytes": int(fbytes), "rank": int(frk),
                "value": round(fbytes / fsecs / 1e9, 4)}
    wall = time.perf_counter() - t0
    val = full["value"] if full else sample_val
    sample = (f"{args.steps} x leading {m}x{cols} column block of the 65536^2 ctr(seed {SEED}) matrix "
              f"(rank {rk}), {tsum / args.steps:.2f} s each, single-threaded gf2::block_iterative_ple")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * (full["seconds"] if full else tsum / args.steps), 3),
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"block_iterative_ple {N_DEFAULT}x{N_DEFAULT} (BASELINE config 5, 1 GPU)",
                   "timed": ("value = ONE full 65536^2 run (the device arm's exact config); the K "
                             "steps are the bounded sample, reported in cpu_baseline.sample_value")
                   if full else "value = the bounded sample (--ref-sample-only)",
                   "generator": "ctr (SURVEY.md 8(d)), oracle/liboracle.so", "seed": SEED,
                   "panel_bits": 64},
        "full_size": full,
        "cpu_baseline": {"value": round(val, 4), "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": sample, "sample_value": round(sample_val, 4),
                         "host_cores": os.cpu_count()},
        "e2e": {"value": round(val, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 2),
    }))


# ------------------------------------------------------------------ GPU leg
def gpu_arm(args, rank, world, local_rank):
    import torch
    import paper_1111_6549_b200 as G

    torch.cuda.set_device(local_rank)
    dev = local_rank
    # an explicit stream: the library calls, the CUDA events and every torch op
    # of the timed region are ordered on it (the legacy default stream is not
    # ordered with the library's non-blocking streams)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    m = n = args.n
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    pristine = G.DeviceMatrix(m, n, device=dev)
    pristine.fill_ctr(SEED, stream=sptr)
    work = G.DeviceMatrix(m, n, device=dev)
    cfg = G.PleConfig(device=dev, stream=sptr)
    cfg_t = G.PleConfig(device=dev, stream=sptr, time_kernels=True)

    clocks = ClockSampler(dev)
    clocks.start()
    # warm-up (also yields the rank / checksum for the parity handle)
    for _ in range(args.warmup):
        work.copy_from(pristine, stream=sptr)
        out = G.block_iterative_ple(work, cfg)
    checksum = work.checksum(stream=sptr) if args.warmup else None

    # ---- timed region: K steps, device-resident inputs ----
    barrier()
    clocks.begin()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    tot_bytes = 0.0
    sweep_bytes = 0.0   # bytes the trailing sweeps move (K = 128 for the super-step driver)
    driver = 1
    trail_ms = 0.0      # device-timestamped trailing-update phases (inside the kernel)
    kern_ms = 0.0       # CUDA-event duration of the persistent PLE kernel
    launches = 0        # persistent-kernel launches (one per PLE)
    kernel_launches = 0
    panel_ms = apply_ms = 0.0
    for _ in range(args.steps):
        work.copy_from(pristine, stream=sptr)
        out = G.block_iterative_ple(work, cfg_t)
        st = out.stats
        tot_bytes += st["alg_bytes"]
        sweep_bytes += st["sweep_bytes"]
        driver = int(st["driver"])
        trail_ms += st["trailing_ms"]
        kern_ms += st["kernel_ms"]
        panel_ms += st["panel_ms"]
        apply_ms += st["coef_ms"]
        launches += 1
        # tile + init + persistent PLE + untile per step
        kernel_launches += 4
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)

    # ---- e2e: drop-in gf2cu_ple on pinned host buffers ----
    Wd = (n + 63) // 64
    host = torch.empty((m, Wd), dtype=torch.int64, pin_memory=True)
    host_np = host.numpy().view(np.uint64)
    pristine.download(host_np)
    src = host_np.copy()
    view = G.MatrixView(host_np, Wd, 0, m, n)
    e2e_steps = max(1, min(args.steps, 3))
    np.copyto(host_np, src)
    G.block_iterative_ple(view, cfg)  # warm the cached device buffers
    barrier()
    e2e_s = 0.0
    e2e_bytes = 0.0
    for _ in range(e2e_steps):
        np.copyto(host_np, src)  # restore the input (host memcpy, outside the timing)
        t0 = time.perf_counter()
        o2 = G.block_iterative_ple(view, cfg)
        e2e_s += time.perf_counter() - t0
        e2e_bytes += o2.stats["alg_bytes"]
    e2e_parity = (o2.rank == out.rank)
    # the same drop-in call on PAGEABLE host memory (what a C++ caller's
    # gf2::BitMatrix, a std::vector, hands the wrapper)
    page_np = np.empty((m, Wd), dtype=np.uint64)
    pview = G.MatrixView(page_np, Wd, 0, m, n)
    np.copyto(page_np, src)
    G.block_iterative_ple(pview, cfg)
    pg_s, pg_bytes, pg_steps = 0.0, 0.0, max(1, min(args.steps, 2))
    for _ in range(pg_steps):
        np.copyto(page_np, src)
        t0 = time.perf_counter()
        o3 = G.block_iterative_ple(pview, cfg)
        pg_s += time.perf_counter() - t0
        pg_bytes += o3.stats["alg_bytes"]
    pg_words = (G.host_checksum(page_np, n) == checksum) if checksum is not None else None
    del page_np, pview
    # the in-place L\E the host received (part of it streamed out while the
    # kernel ran) against the device-resident run's result
    e2e_words = (G.host_checksum(host_np, n) == checksum) if checksum is not None else None

    # ---- max over ranks ----
    vals = torch.tensor([dev_ms, tot_bytes, e2e_s, e2e_bytes, kern_ms, float(launches)],
                        dtype=torch.float64, device="cuda")
    if dist is not None:
        allv = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(allv, vals)
        allv = torch.stack(allv).cpu().numpy()
    else:
        allv = vals.cpu().numpy()[None, :]
    max_ms = float(allv[:, 0].max())
    sum_bytes = float(allv[:, 1].sum())
    e2e_max_s = float(allv[:, 2].max())
    e2e_sum_bytes = float(allv[:, 3].sum())

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    value = sum_bytes / (max_ms * 1e-3) / 1e9
    e2e_value = e2e_sum_bytes / e2e_max_s / 1e9
    peak, peak_kind = load_peaks()
    # algorithmic bytes = SURVEY.md 8(d)'s per-unit figure (one read + one write
    # of every trailing tail word per 64-column panel step) x the steps of one
    # launch. The super-step driver sweeps two panels per pass, so the bytes it
    # actually moves (sweep_bytes, and the ncu DRAM traffic) are about half.
    per_launch_bytes = tot_bytes / max(1, launches)
    per_launch_sweep = sweep_bytes / max(1, launches)
    per_launch_ms = kern_ms / max(1, launches)
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else None
    traffic_ratio = load_traffic(driver)
    super_step = driver == 2
    cap = load_capture(driver)
    dram_phys = None
    if cap.get("dram_bytes_read") and cap.get("duration_ms_under_ncu"):
        dram_phys = ((cap["dram_bytes_read"] + cap["dram_bytes_write"]) / (cap["duration_ms_under_ncu"] * 1e-3)
                     / 1e9 / peak)
    roofline = {
        # The limiter is the L1TEX data pipe (Gray-table lookups in shared
        # memory + the global load/store), not DRAM: `frac` is the metric's
        # EFFECTIVE figure (K = 64 algorithmic bytes over the HBM peak); the
        # physical DRAM use and the L1TEX load come from the committed capture.
        "kernel": "ple_super_kernel" if super_step else "ple_persistent_kernel", "bound": "l1tex",
        "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": (round(per_launch_bytes * traffic_ratio) if traffic_ratio else None),
        "frac_kind": "effective (SURVEY 8(d) K=64 algorithmic bytes / measured HBM peak)",
        "dram_frac_physical": round(dram_phys, 4) if dram_phys else None,
        "l1tex_pct": cap.get("l1tex_throughput_pct_of_peak_active"),
        "capture": cap.get("source"),
        "alg_bytes_per_launch": round(per_launch_bytes),
        "panel_columns_per_sweep": 128 if super_step else 64,
        "sweep_bytes_per_launch": round(per_launch_sweep),
        "sweep_GBps": round(per_launch_sweep / (per_launch_ms * 1e-3) / 1e9, 1) if per_launch_ms else None,
        "limiter": ("L1TEX data pipe: Gray-table lookups (16 B of shared memory per byte of row "
                    "per panel) + the global load/store; see profiles/README.md"),
        "avg_launch_ms": round(per_launch_ms, 4),
        "peak_source": (f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                        else "fallback 6.65 TB/s"),
        "share_of_step": round(kern_ms / max(1e-9, dev_ms), 4),
        # worker 0's device timestamps: rest sweep / panel CTA busy (overlapped
        # with the sweep) / pre-work chunks (apply + look-ahead tiles) + step barrier
        "phases_ms_per_launch": {"trailing_sweep": round(trail_ms / max(1, launches), 3),
                                 "panel_factor_overlapped": round(panel_ms / max(1, launches), 3),
                                 "prework_and_step_barrier": round(apply_ms / max(1, launches), 3)},
        "trailing_sweep_GBps": round(per_launch_bytes / (trail_ms / max(1, launches) * 1e-3) / 1e9, 1)
        if trail_ms > 0 else None,
    }

    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            secs, b, rk = run_reference_sample(n, REF_SAMPLE_COLS, SEED)
            cpu = {"value": round(b / secs[0] / 1e9, 3), "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"leading {n}x{REF_SAMPLE_COLS} column block of the same matrix "
                             f"(rank {rk}), {secs[0]:.2f} s, single-threaded gf2::block_iterative_ple",
                   "host_cores": os.cpu_count()}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(max_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"block_iterative_ple {m}x{n} (BASELINE config 5, 1 GPU)",
                   "generator": "ctr (SURVEY.md 8(d))", "seed": SEED, "rank": int(out.rank),
                   "panel_bits": 64, "panels_per_sweep": 2 if driver == 2 else 1,
                   "parallelism": f"replicas x{world}" if world > 1 else "single",
                   "l2": "input 512 MiB > 126 MB L2; pristine copy restored each step (counted)",
                   "checksum": hex(checksum) if checksum is not None else None},
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(m * Wd * 8), "d2h_bytes_per_step": int(m * Wd * 8),
                "steps": e2e_steps, "ms_per_step": round(1e3 * e2e_max_s / e2e_steps, 3),
                "rank_matches_device_run": bool(e2e_parity),
                "output_matches_device_run": e2e_words,
                "host_memory": "pinned (torch pin_memory)",
                "streamed_input": {"row_blocks": int(o2.stats["input_blocks"]),
                                   "first_block_rows": int(o2.stats["input_first_rows"]),
                                   "super_steps_before_last_block": int(o2.stats["input_first_steps"])},
                "pageable": {"value": round(pg_bytes / pg_s / 1e9, 2), "unit": UNIT, "steps": pg_steps,
                             "ms_per_step": round(1e3 * pg_s / pg_steps, 3),
                             "output_matches_device_run": pg_words}},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": int(kernel_launches),
    }
    print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


N_SCALE = 131072


def scale_n(world: int, n_arg: int) -> int:
    """The N > 1 workload: BASELINE config 5's 131072^2 at every N (strong
    scaling, north_star: "near-linear row-slab scaling to 8 GPUs on
    131072x131072"); --size overrides it."""
    return n_arg if n_arg != N_DEFAULT else (N_SCALE if world > 1 else N_DEFAULT)


def q_to_bytes(m, n, q):
    W = (n + 63) // 64
    q = np.asarray(q, dtype=np.int64)
    rh, rbh, r = [], [], 0
    for w in range(W):
        rb = int(np.count_nonzero((q >= 64 * w) & (q < 64 * w + 64)))
        rh.append(r)
        rbh.append(rb)
        r += rb
    return alg_bytes_from_history(m, n, rh, rbh)


def gpu_sharded_arm(args, rank, world, local_rank):
    """N > 1: the row-sharded PLE (paper_1111_6549_b200/shard.py), one process
    per GPU over NCCL, on 131072^2 (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_1111_6549_b200 import shard as S

    torch.cuda.set_device(local_rank)
    if "RANK" not in os.environ:  # --sharded at N=1 without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        os.environ["RANK"], os.environ["WORLD_SIZE"] = "0", "1"
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    n = scale_n(world, args.n)
    m = n
    eng = S.GpuShardEngine(m, n, rank, world, block=256, device=local_rank)

    def one():
        eng.fill_ctr(SEED)
        return S.run_sharded(eng, dist)

    res = None
    for _ in range(args.warmup):
        res = one()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.begin()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with eng.stream_ctx():
        ev0.record()
        for _ in range(args.steps):
            res = one()
        ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)
    bytes_per_step = float(q_to_bytes(m, n, res.q))
    # e2e: each rank's rows in from pinned host memory, L\E rows back out
    Wd = (n + 63) // 64
    host_in = torch.empty((max(1, eng.m_local), Wd), dtype=torch.int64, pin_memory=True)
    eng.fill_ctr(SEED)
    eng.download(host_in.numpy().view(np.uint64))
    t_e2e = 0.0
    e2e_steps = max(1, min(args.steps, 2))
    for _ in range(e2e_steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.upload(host_in.numpy().view(np.uint64)[: eng.m_local])
        out2 = S.run_sharded(eng, dist)  # finish() downloads this rank's rows
        torch.cuda.synchronize()
        t_e2e += time.perf_counter() - t0
        assert out2.rank == res.rank
    vals = torch.tensor([dev_ms, t_e2e], dtype=torch.float64, device="cuda")
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    max_ms, e2e_max_s = float(vals[0]), float(vals[1])
    if rank == 0:
        value = bytes_per_step * args.steps / (max_ms * 1e-3) / 1e9
        peak, peak_kind = load_peaks()
        per_gpu = value / world
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"block_iterative_ple {m}x{n} row-sharded over {world} GPUs "
                                   f"(BASELINE config 5, strong scaling: the same matrix at every N)",
                       "generator": "ctr (SURVEY.md 8(d))", "seed": SEED, "rank": int(res.rank),
                       "panel_bits": 64, "parallelism": f"row-sharded x{world} (block-cyclic 256-row blocks, NCCL)",
                       "l2": "per-GPU shard > 126 MB L2"},
            "e2e": {"value": round(bytes_per_step * e2e_steps / e2e_max_s / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(m * Wd * 8), "d2h_bytes_per_step": int(m * Wd * 8),
                    "steps": e2e_steps},
            "roofline": {"kernel": "sharded step sequence (per GPU)", "bound": "hbm",
                         "achieved": round(per_gpu, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_gpu / peak, 4), "traffic": None,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
            "cpu_baseline": None,
            "clocks": clk,
            "gpu_launches": None,
        }))
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def gpu_peer_arm(args, rank, world, local_rank):
    """N > 1 (default): the device-driven row-sharded PLE (peer.py, kernel
    csrc/ple_peer.cuh): one process and ONE persistent kernel per GPU for the
    whole factorization, the ranks exchanging the panel column and pivot-row
    tails through NVLink peer memory (CUDA IPC) with device-side counters --
    no host call or collective per step. Strong scaling on BASELINE config
    5's 131072^2."""
    import torch
    import torch.distributed as dist
    from paper_1111_6549_b200.peer import PeerEngine, exchange_handles

    torch.cuda.set_device(local_rank)
    if "RANK" not in os.environ:  # --sharded at N=1 without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29563")
        os.environ["RANK"], os.environ["WORLD_SIZE"] = "0", "1"
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    n = scale_n(world, args.n)
    m = n
    stream = torch.cuda.current_stream()
    eng = PeerEngine(m, n, rank, world, block=256, device=local_rank, stream=stream.cuda_stream)
    exchange_handles(eng, dist)
    kernel_ms = []

    def one():
        eng.fill_ctr(SEED)  # the input, regenerated on the device (counted)
        eng.reset()
        dist.barrier()
        st = eng.run()
        # no rank resets for the next run before every kernel is done (the
        # last step's signals into the peers' counters have landed)
        dist.barrier()
        kernel_ms.append(st["kernel_ms"])
        return st

    st = None
    for _ in range(args.warmup):
        st = one()
    kernel_ms.clear()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.begin()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        st = one()
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)
    res = eng.finish()
    bytes_per_step = float(st["alg_bytes"])
    # e2e: each rank's rows in from pinned host memory, its L\E rows back out
    Wd = (n + 63) // 64
    host_in = torch.empty((max(1, eng.m_local), Wd), dtype=torch.int64, pin_memory=True)
    eng.fill_ctr(SEED)
    host_in_np = host_in.numpy().view(np.uint64)
    eng.download(host_in_np)
    t_e2e = 0.0
    e2e_steps = max(1, min(args.steps, 2))
    for _ in range(e2e_steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.upload(host_in_np[: eng.m_local])
        eng.reset()
        dist.barrier()
        eng.run()
        dist.barrier()
        out2 = eng.finish()  # replicated outcome + this rank's rows to the host
        torch.cuda.synchronize()
        t_e2e += time.perf_counter() - t0
        assert out2.rank == res.rank
    vals = torch.tensor([dev_ms, t_e2e, max(kernel_ms), statistics.median(kernel_ms)],
                        dtype=torch.float64, device="cuda")
    allv = [torch.zeros_like(vals) for _ in range(world)]
    dist.all_gather(allv, vals)
    allv = torch.stack(allv).cpu().numpy()
    max_ms, e2e_max_s, kmax = float(allv[:, 0].max()), float(allv[:, 1].max()), float(allv[:, 2].max())
    per_rank = [{"rank": i, "device_ms": round(float(allv[i, 0]), 3),
                 "kernel_ms_median": round(float(allv[i, 3]), 3), "kernel_ms_max": round(float(allv[i, 2]), 3)}
                for i in range(world)]
    print(f"[bench rank {rank}/{world}] device {torch.cuda.get_device_name(local_rank)} "
          f"kernel_ms median {statistics.median(kernel_ms):.3f} max {max(kernel_ms):.3f}", file=sys.stderr)
    if rank == 0:
        value = bytes_per_step * args.steps / (max_ms * 1e-3) / 1e9
        peak, peak_kind = load_peaks()
        per_gpu_kernel = bytes_per_step / world / (kmax * 1e-3) / 1e9
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"block_iterative_ple {m}x{n} row-sharded over {world} GPUs "
                                   f"(BASELINE config 5, strong scaling: the same matrix at every N)",
                       "generator": "ctr (SURVEY.md 8(d))", "seed": SEED, "rank": int(res.rank),
                       "panel_bits": 64,
                       "parallelism": f"row-sharded x{world} (block-cyclic 256-row blocks), one persistent "
                                      "kernel per GPU, NVLink peer-memory exchange (ple_peer.cuh)",
                       "l2": "per-GPU shard > 126 MB L2; input regenerated on the device each step (counted)"},
            "e2e": {"value": round(bytes_per_step * e2e_steps / e2e_max_s / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(m * Wd * 8), "d2h_bytes_per_step": int(m * Wd * 8),
                    "steps": e2e_steps},
            "roofline": {"kernel": "ple_peer_kernel", "bound": "hbm",
                         "achieved": round(per_gpu_kernel, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_gpu_kernel / peak, 4), "traffic": None,
                         "avg_launch_ms": round(kmax, 3),
                         "note": "per GPU: the matrix's algorithmic bytes / N over the slowest rank's kernel",
                         "per_rank": per_rank,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
            "cpu_baseline": None,
            "clocks": clk,
            "gpu_launches": 4 * args.steps,
        }))
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-sample-only", action="store_true",
                    help="--impl reference: skip the full-size 65536^2 run (value = the sample)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded PLE even at N=1 (testing)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent single-GPU replicas instead of the row-sharded PLE")
    ap.add_argument("--host-sharded", action="store_true",
                    help="the host-orchestrated row-sharded path (shard.py, NCCL collectives per "
                         "step) instead of the device-driven one (peer.py)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    if (world > 1 and not args.replicas) or args.sharded:
        if args.host_sharded:
            gpu_sharded_arm(args, rank, world, local_rank)
        else:
            gpu_peer_arm(args, rank, world, local_rank)
        return
    gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
