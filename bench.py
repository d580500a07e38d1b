"""Benchmark of the hot path (BASELINE.json metric): relit vertices/s (and shifted Haar coefficients
/s) on config c5 -- 6 x 256 x 256 cube-map light, 64 light/rotation frames, 1M vertices with
6 x 1024-coefficient transfer vectors -- as a fraction of the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

One step = the whole hot path over one batch:
  (a0-a5) haar_shift_coeffs: 64 frames x 6 faces of 256x256 Haar pyramids shifted in the Haar
          domain (rank 0; N=1: full pyramids written, the relight reads their band in place;
          N>1: band written, then NCCL-broadcast);
  (a6)    relight_vertices: R[v][b] = <T_v, L'_b band> for this rank's vertex rows;
  (e)     N>1: radiance gathered to rank 0 in chunks overlapped with the relight.
Inputs are resident in HBM when timing starts; T (24.6 GB) is streamed every step, so the working
set is far larger than L2 (no flush needed).  Rank 0 prints ONE JSON line.

--impl reference times the fp64 CPU oracle (oracle/, test infrastructure) on this host's cores on
a bounded sample of the same workload (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "relit_vertices_per_sec"
UNIT = "vertices/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0     # GB/s, B200_PROFILING.md fallback
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c5")
    p.add_argument("--vertices", type=int, default=None, help="override V (debug only)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--chunks", type=int, default=4)
    p.add_argument("--e2e-chunks", type=int, default=4)
    p.add_argument("--no-graph", action="store_true", help="c2: direct launches instead of a CUDA graph")
    p.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                   help="N>1: fused relight + gather into rank 0's buffer over NVLink (p2p) or NCCL gather")
    p.add_argument("--start-level", type=int, default=None,
                   help="coarse-start shift (row f4, approximate): shift the level-L approximation only")
    return p.parse_args()


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# fp64 ALU roofline of the rotation (row f1): peak = 148 SMs x 64 fp64 FMA per clock
# (one warp DFMA per 2 cycles per SMSP, consistent with ncu's fp64-pipe counters on the shift
# kernels) x 2 flops x the max SM clock; the algorithmic count per rotated pixel: the chain rule
# (1.63 rotated samples x ~63 flops: the rotation, |(x', z')| and two atan2; 2 output differences x
# ~31 flops: two bilinear field samples and the increments) plus the bottom-up (~20 per pixel).
ROT_FP64_FLOPS_PER_PIXEL = 185


def fp64_peak_tflops():
    mhz = 1965.0
    try:
        with open(PEAKS_PATH) as fh:
            mhz = float(json.load(fh).get("sm_max_mhz", mhz))
    except (OSError, ValueError):
        pass
    return 148 * 64 * 2 * mhz * 1e6 / 1e12, f"derived: 148 SMs x 64 fp64 FMA/clk x 2 x {mhz:.0f} MHz (DESIGN.md §5.9)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms on a background
    thread; ``mark(True/False)`` brackets the timed region and ``summary()`` reports the samples
    taken inside it (the nvidia-smi CLI cannot sample a region this short)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (t, sm_mhz, reasons_mask, in_region)
        self.in_region = False
        self.stop = False
        self.thread = None
        self.max_mhz = None
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def _run(self):
        nv, h = self.nv, self.h
        while not self.stop:
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                mask = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((time.perf_counter(), mhz, mask, self.in_region))
            except Exception as e:  # pragma: no cover
                self.err = repr(e)
                return
            time.sleep(0.002)

    def mark(self, inside: bool):
        self.in_region = inside

    def __exit__(self, *exc):
        self.stop = True
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        inside = [s for s in self.samples if s[3]]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "error": self.err}
        reasons = set()
        for _, _, mask, _ in inside:
            for bit, name in REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in inside]), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside), "source": "nvml, 2 ms poll"}


# ------------------------------------------------------------------------------------ oracle arm

def oracle_sample(cfg, den=16, seed_off=0):
    """Time the fp64 oracle on 1/den of the step's workload: the shift of frames/den frames (at
    least one) and the relight of vertices/den vertex rows x all frames.  Returns (measured
    seconds, vertices in the sample, description).  The sample rate (sample vertices / measured
    time) equals the full step's rate when the oracle scales linearly in frames and rows; nothing
    is extrapolated into the reported step time."""
    from oracle import relight as orelight
    from oracle import shift as oshift
    N, F, kf = 1 << cfg.log2n, cfg.faces, cfg.k_face
    frames_s = max(1, cfg.frames // den)
    rows_s = max(1, cfg.vertices // den)
    light = synth.light_pyramids(cfg.seed, frames_s, F, cfg.log2n)
    s = synth.c5_shifts(cfg.seed, cfg.frames, cfg.log2n)[:frames_s]
    sh = np.broadcast_to(s[:, None, :], (frames_s, F, 2))
    if cfg.name == "c5t":
        rows = (synth.shading_rows(cfg.seed, seed_off, rows_s, F, kf, synth.STREAM_BRDF),
                synth.shading_rows(cfg.seed, seed_off, rows_s, F, kf, synth.STREAM_VIS))
    else:
        rows = (synth.transfer_rows(cfg.seed, seed_off, rows_s, F, kf),)
    t0 = time.perf_counter()
    shifted = oshift.shift_coeffs(light, sh, 2)
    t_shift = time.perf_counter() - t0
    Lb = np.concatenate([shifted] * (cfg.frames // frames_s + 1))[: cfg.frames]
    t0 = time.perf_counter()
    if cfg.name == "c5t":
        orelight.relight_triple(rows[0], rows[1], Lb, F, kf)
    else:
        orelight.relight(rows[0], Lb, F, kf)
    t_rel = time.perf_counter() - t0
    what = "triple product" if cfg.name == "c5t" else "relight"
    desc = (f"oracle fp64 on 1/{den} of the step, measured (not extrapolated): shift of {frames_s}/{cfg.frames} "
            f"frames x {F} faces of {N}x{N} ({t_shift:.3f}s) + {what} of {rows_s}/{cfg.vertices} vertex rows x "
            f"{cfg.frames} frames ({t_rel:.3f}s); value = sample vertices / measured time")
    return t_shift + t_rel, rows_s, desc


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        blas = [i for i in info if i.get("user_api") == "blas"]
        if blas:
            return int(blas[0].get("num_threads", 1))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    warm, steps = max(args.warmup, 0), max(args.steps, 1)
    ref_den = 256 if cfg.name == "c5t" else 16     # the triple-product oracle is ~60x slower per vertex
    times = []
    for i in range(warm + steps):
        t, rows_s, desc = oracle_sample(cfg, ref_den, seed_off=(i * 997) % max(1, cfg.vertices))
        if i >= warm:
            times.append(t)
    t = statistics.median(times)
    value = rows_s / t
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "step": f"1/{ref_den} of the workload per step ({rows_s} vertices); ms_per_step is that measured sample step",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(cfg, gpus):
    N = 1 << cfg.log2n
    return {"workload": f"{cfg.name}: {cfg.faces}x{N}x{N} cube-map light, {cfg.frames} frames, "
                        f"{cfg.vertices} vertices, transfer {cfg.faces}x{cfg.k_face} coefficients",
            "faces": cfg.faces, "N": N, "frames": cfg.frames, "vertices": cfg.vertices, "k_face": cfg.k_face,
            "parallelism": f"dp{gpus} over vertex rows", "l2": "no flush: transfer matrix streamed every step "
            f"({cfg.vertices * cfg.faces * cfg.k_face * 4 / 1e9:.1f} GB) >> 126 MB L2"}


# ------------------------------------------------------------------------------------ our arm

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200 import dist as hsdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    V = args.vertices or cfg.vertices
    n, F, B, kf = cfg.log2n, cfg.faces, cfg.frames, cfg.k_face
    N = 1 << n
    K = F * kf
    r0, rows = hsdist.shard_rows(V, world, rank)

    # ---- inputs resident in HBM (untimed)
    T = torch.empty((rows, K), dtype=torch.float32, device=dev)
    hs.hs_fill_transfer(T, r0, F, kf, cfg.seed, synth.STREAM_T)
    light_np = synth.light_pyramids(cfg.seed, B, F, n)
    shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
    light = torch.from_numpy(light_np).to(dev)
    full_out = world == 1
    shifted = torch.empty((B, F, N * N if full_out else kf), dtype=torch.float32, device=dev)
    ws = torch.empty(hs.haar_shift_workspace_bytes(2, n, F, B), dtype=torch.uint8, device=dev)
    shifted_band = torch.empty((B, F, kf), dtype=torch.float32, device=dev) if args.start_level is not None else None
    if args.start_level is not None and world > 1:
        raise SystemExit("--start-level is a single-GPU option")
    R = torch.empty((rows, B), dtype=torch.float32, device=dev)
    R_full = torch.empty((V, B), dtype=torch.float32, device=dev) if (rank == 0 and world > 1) else None
    fs0, fsn = hsdist.shard_rows(B, world, rank)          # this rank's frames of the sharded shift
    band_local = torch.empty((fsn, F, kf), dtype=torch.float32, device=dev) if world > 1 else None
    if world > 1:
        ws = torch.empty(max(1, hs.haar_shift_workspace_bytes(2, n, F, max(fsn, 1))), dtype=torch.uint8, device=dev)
    gather_mode = args.gather if world > 1 else "none"
    R_view = None
    fence_flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if gather_mode == "p2p":
        # fused relight + gather: every rank's relight epilogue stores straight into rank 0's buffer
        try:
            R_view = hsdist.open_peer_view(R_full, (V, B), dev)
        except Exception as e:  # devices cannot reach each other: NCCL gather instead
            if rank == 0:
                print(f"[bench] p2p gather unavailable ({e!r}); using the NCCL gather", file=sys.stderr)
            gather_mode = "nccl"
        ok = torch.tensor([1 if R_view is not None or rank == 0 else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            gather_mode = "nccl"
    rws_bytes = hs.relight_workspace_bytes(F, kf, B)
    rws = torch.empty(rws_bytes + 1024, dtype=torch.uint8, device=dev) if rws_bytes else None
    if rws is not None:
        rws = rws[(-rws.data_ptr()) % 1024:]
    stream = torch.cuda.current_stream()
    launches = {"n": 0}
    rel_events = []
    shift_events = []

    def relight_fn(Tc, band, Rc):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hs.relight_vertices(Tc, band, F, kf, out=Rc, workspace=rws)
        e1.record(stream)
        launches["n"] += hs.last_launch_count()
        rel_events.append((e0, e1, Tc.shape[0]))

    def step():
        """One pass of the hot path; returns this rank's result tensor (R, or R_full on rank 0)."""
        if world > 1:
            # shift sharded by frame, band all-gathered over NVLink
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hs.haar_shift_coeffs(light[fs0:fs0 + fsn], shifts[fs0:fs0 + fsn], 2, cfg.band_levels, out=band_local,
                                 workspace=ws)
            e1.record(stream)
            shift_events.append((e0, e1))
            launches["n"] += hs.last_launch_count()
            hsdist.allgather_band(band_local, shifted)
            if gather_mode == "p2p":
                hsdist.relight_into_peer(T, shifted, V, relight_fn, R_view)
                hsdist.rows_landed_fence(fence_flag)   # stream-ordered: rank 0's later work sees every row
                return R_full
            _, full = hsdist.relight_and_gather(T, shifted, V, relight_fn, R_full, chunks=args.chunks)
            return full
        if rank == 0:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if args.start_level is not None:
                hs.haar_shift_coeffs_coarse(light, shifts, args.start_level, cfg.band_levels, out=shifted_band,
                                            workspace=ws)
            else:
                hs.haar_shift_coeffs(light, shifts, 2, n if full_out else cfg.band_levels, out=shifted, workspace=ws)
            e1.record(stream)
            shift_events.append((e0, e1))
            launches["n"] += hs.last_launch_count()
        relight_fn(T, shifted_band if args.start_level is not None else shifted, R)
        return R

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches["n"] = 0
    rel_events.clear()
    shift_events.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    rel_ms = [a.elapsed_time(b) for a, b, _ in rel_events]
    rel_rows = [r for _, _, r in rel_events]
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    gpu_launches = launches["n"]

    # ---- dominant kernel roofline (relight): algorithmic bytes per launch / average launch time
    peak, peak_src = hbm_peak()
    bytes_per_row = K * 4 + B * 4
    alg_bytes = [r * bytes_per_row + B * K * 4 for r in rel_rows]
    avg_ms = sum(rel_ms) / len(rel_ms)
    achieved = (sum(alg_bytes) / len(alg_bytes)) / (avg_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"{cfg.name}:relight_b{B}") if (V == cfg.vertices and world == 1) else None
    except Exception:
        pass

    # ---- end to end through the public API with host buffers (pinned), N GPUs
    e2e = None
    if not args.no_e2e and world == 1:
        # pipelined host-buffer path (paper_1705_07272_b200.pipeline): per step the 64 pyramids go
        # host -> device and the full radiance device -> host, overlapped with the compute
        from paper_1705_07272_b200.pipeline import ShiftRelightPipeline
        light_h = torch.from_numpy(light_np).pin_memory()
        Rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        pipe = ShiftRelightPipeline(T, F, n, B, cfg.band_levels, chunks=args.e2e_chunks, full_pyramids=True)
        for _ in range(max(1, args.warmup)):
            pipe.step(light_h, shifts, Rh)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            ev = pipe.step(light_h, shifts, Rh)
        stream.wait_event(ev)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        e2e = {"value": V / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(light_np.nbytes),
               "d2h_bytes_per_step": int(V * B * 4), "ms_per_step": e_ms,
               "note": "ShiftRelightPipeline.step per step: pinned H2D of the 64 light pyramids, shift, chunked "
                       f"relight ({args.e2e_chunks} chunks) with each chunk's radiance D2H overlapped; T is scene "
                       "data resident in HBM"}
    elif not args.no_e2e:
        # N > 1 host buffers: each rank H2Ds its own frames, shifts them, the band is all-gathered,
        # and each rank D2Hs its own radiance rows, chunked under its relight, into ONE shared
        # page-locked host array (all N PCIe links carry the gather)
        from paper_1705_07272_b200.pipeline import ShardedShiftRelightPipeline
        light_h = torch.from_numpy(light_np).pin_memory()
        shared = hsdist.SharedHostBuffer((V, B))
        pipe = ShardedShiftRelightPipeline(T, F, n, B, cfg.band_levels, V, chunks=args.e2e_chunks)
        for _ in range(max(1, args.warmup)):
            pipe.step(light_h, shifts, shared.tensor)
        torch.cuda.synchronize()
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            ev = pipe.step(light_h, shifts, shared.tensor)
        stream.wait_event(ev)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        dist.barrier()
        if rank == 0:   # the shared host array holds every rank's rows: spot-check against one rank's device rows
            ok = bool(torch.equal(shared.tensor[: pipe.R.shape[0]], pipe.R.cpu()))
        shared.close()
        bytes_io = torch.tensor([pipe.h2d_bytes(), pipe.d2h_bytes()], dtype=torch.float64, device=dev)
        dist.all_reduce(bytes_io)
        e2e = {"value": V / (float(e_ms.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(bytes_io[0].item()), "d2h_bytes_per_step": int(bytes_io[1].item()),
               "ms_per_step": float(e_ms.item()),
               "note": "ShardedShiftRelightPipeline.step per step on every rank: pinned H2D of the rank's own "
                       "light frames, sharded shift, band all-gather (NCCL), chunked relight of the rank's rows "
                       "with each chunk's D2H into one shared page-locked host array (bytes summed over ranks); "
                       "T is scene data resident in HBM"}
        if rank == 0:
            e2e["rank0_rows_match_device"] = ok

    if rank == 0:
        line = {
            "metric": METRIC, "value": V / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "arithmetic": "fp32 in / out; shift fields fp64; relight: fp32 GEMV (B <= 8) or tcgen05 products of "
                          "fp16 hi/lo splits accumulated in fp32 (B % 64 == 0), within 1e-5 of the fp64 oracle",
            "config": workload_config(cfg, world),
            "gather": gather_mode,
            "vertex_frames_per_sec": V * B / (ms_max * 1e-3),
            "shift_coeffs_per_sec": (B * F * N * N / (statistics.median([a.elapsed_time(b) for a, b in shift_events])
                                                       * 1e-3)) if shift_events else None,
            "roofline": {"bound": "hbm", "kernel": "relight_vertices", "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": sum(alg_bytes) / len(alg_bytes),
                         "avg_launch_ms": avg_ms, "share_of_step": sum(rel_ms) / args.steps / ms},
            "shift_ms": (sum(a.elapsed_time(b) for a, b in shift_events) / len(shift_events)) if shift_events else None,
            "shift_start_level": args.start_level,
            "shift_frac_hbm": ((2 * B * F * N * N * 4 if full_out else fsn * F * (N * N + kf) * 4) /
                               (sum(a.elapsed_time(b) for a, b in shift_events) / len(shift_events) * 1e-3) / 1e9 / peak)
            if shift_events else None,
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            # a few seconds of fp64 work: 1/4 of the step at K = 6144, less for longer transfer rows
            den = 4 * max(1, (cfg.faces * cfg.k_face) // 6144)
            t_s, rows_s, desc = oracle_sample(cfg, den)
            line["cpu_baseline"] = {"value": rows_s / t_s, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                                    "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_aux(args, cfg):
    """Configs c2 (32x32, 1 shift, 1k vertices), c3 (6x64x64, 10k vertices, one frame per step:
    global 1-degree azimuth rotation + relight) and c4 (6x128x128, 100k vertices, per-vertex shifts,
    fused relight_vertices_shifted).  One GPU (N > 1: vertex rows sharded, no gather)."""
    import torch
    import torch.distributed as dist

    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200 import dist as hsdist
    from oracle import relight as orelight
    from oracle import shift as oshift

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    V = args.vertices or cfg.vertices
    n, F = cfg.log2n, cfg.faces
    N = 1 << n
    kf = cfg.k_face
    K = F * kf
    r0, rows = hsdist.shard_rows(V, world, rank)
    stream = torch.cuda.current_stream()
    T = torch.empty((rows, K), dtype=torch.float32, device=dev)
    hs.hs_fill_transfer(T, r0, F, kf, cfg.seed, synth.STREAM_T)
    light_np = synth.light_pyramids(cfg.seed, 1, F, n)
    light = torch.from_numpy(light_np).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if cfg.name == "c2" else None
    launches = {"n": 0}
    dom = []  # (event0, event1) around the dominant call
    if cfg.name == "c4":
        sv_np = synth.c4_vertex_shifts(cfg.seed, V, n)
        sv = torch.from_numpy(sv_np[r0:r0 + rows].copy()).to(dev)
        L0 = light[0]
        R = torch.empty((rows,), dtype=torch.float32, device=dev)
        ws = torch.empty(hs.relight_shifted_workspace_bytes(rows, F, n), dtype=torch.uint8, device=dev)
        kernel_name = "relight_vertices_shifted (shift + dot)"
        alg_bytes = rows * (K * 4 + 8 + 4) + F * N * N * 4

        def step(i):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hs.relight_vertices_shifted(T, L0, sv, out=R, workspace=ws)
            e1.record(stream)
            dom.append((e0, e1))
            launches["n"] += hs.last_launch_count()
            return R
    else:
        frames = synth.c3_shifts(n, 360) if cfg.name == "c3" else np.array([[3.25, 7.5]])
        shifted = torch.empty((1, F, N * N), dtype=torch.float32, device=dev)
        R = torch.empty((rows, 1), dtype=torch.float32, device=dev)
        ws = torch.empty(max(1, hs.haar_shift_workspace_bytes(2, n, F, 1)), dtype=torch.uint8, device=dev)
        kernel_name = "relight_vertices (GEMV, batch 1)"
        alg_bytes = rows * (K * 4 + 4) + K * 4

        def step(i):
            s = np.broadcast_to(frames[i % len(frames)][None, None, :], (1, F, 2))
            hs.haar_shift_coeffs(light, s, 2, out=shifted, workspace=ws)
            launches["n"] += hs.last_launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hs.relight_vertices(T, shifted, F, kf, out=R)
            e1.record(stream)
            dom.append((e0, e1))
            launches["n"] += hs.last_launch_count()
            return R

        # c3, device-resident loop: the frames are independent, so the (latency-bound, 6-CTA)
        # shift of frame i+1 runs on a side stream under the HBM-bound relight of frame i
        # (double-buffered band); every frame still gets its own shift and relight
        sstream = torch.cuda.Stream(dev)
        shifted2 = [shifted, torch.empty_like(shifted)]
        ws2 = [ws, torch.empty_like(ws)]
        ev_shift = [torch.cuda.Event(), torch.cuda.Event()]
        ev_rel = [torch.cuda.Event(), torch.cuda.Event()]
        pipe = {"next": None}

        def enqueue_shift(i):
            b = i & 1
            s = np.broadcast_to(frames[i % len(frames)][None, None, :], (1, F, 2))
            sstream.wait_event(ev_rel[b])                 # the relight that read this buffer is done
            hs.haar_shift_coeffs(light, s, 2, out=shifted2[b], workspace=ws2[b], stream=sstream)
            launches["n"] += hs.last_launch_count()
            ev_shift[b].record(sstream)
            pipe["next"] = i

        def step_pipelined(i):
            b = i & 1
            if pipe["next"] != i:
                enqueue_shift(i)
            stream.wait_event(ev_shift[b])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hs.relight_vertices(T, shifted2[b], F, kf, out=R)
            e1.record(stream)
            ev_rel[b].record(stream)
            dom.append((e0, e1))
            launches["n"] += hs.last_launch_count()
            enqueue_shift(i + 1)
            return R

    def timed(fn, i, evs):
        """c2 fits in L2: flush it before every step, outside the step's own (start, end) events"""
        if flush is None:
            return fn(i)
        flush.zero_()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        out = fn(i)
        b_.record(stream)
        evs.append((a_, b_))
        return out

    graph = None
    if cfg.name == "c2" and not args.no_graph:
        # c2 is launch-latency bound: capture one step (shift + relight, fixed shift) in a CUDA graph
        # after the warm-up and replay it; the L2 flush stays outside the graph and outside the timing
        def step_graph(i):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            dom.append((e0, e1))
            launches["n"] += graph_launches
            return R

    step_ev = []
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if cfg.name == "c2" and not args.no_graph:
        s_cap = torch.cuda.Stream(dev)
        s_cap.wait_stream(stream)
        n0 = launches["n"]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s_cap):
            sh0 = np.broadcast_to(frames[0][None, None, :], (1, F, 2))
            hs.haar_shift_coeffs(light, sh0, 2, out=shifted, workspace=ws)
            launches["n"] += hs.last_launch_count()
            hs.relight_vertices(T, shifted, F, kf, out=R)
            launches["n"] += hs.last_launch_count()
        graph_launches = launches["n"] - n0
        kernel_name = f"shift + relight (one CUDA graph replay: {graph_launches} kernels)"
        stream.wait_stream(s_cap)
        for i in range(2):
            graph.replay()
        torch.cuda.synchronize()
        step = step_graph
    launches["n"] = 0
    dom.clear()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for i in range(args.steps):
            timed(step_pipelined if cfg.name == "c3" else step, i, step_ev)
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    timed_launches = launches["n"]
    if flush is not None:   # c2: the timed steps exclude the L2 flush that precedes each of them
        ms = sum(a_.elapsed_time(b_) for a_, b_ in step_ev) / len(step_ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    dom_ms = sum(a.elapsed_time(b) for a, b in dom) / len(dom)
    peak, peak_src = hbm_peak()
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    e2e = None
    if not args.no_e2e:
        light_h = torch.from_numpy(light_np).pin_memory()
        Rh = torch.empty(R.shape, dtype=torch.float32).pin_memory()

        def e2e_step(i):
            light.copy_(light_h, non_blocking=True)
            Rh.copy_(step(i), non_blocking=True)

        if cfg.name == "c3":
            # per frame: H2D of the light into a double buffer (copy stream), the shift on the side
            # stream, the relight, and the radiance D2H (second copy stream) into alternating pinned
            # buffers -- frame i+1's copy and shift run under frame i's relight
            cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            lbuf = [torch.empty_like(light), torch.empty_like(light)]
            rbuf = [torch.empty_like(R), torch.empty_like(R)]
            rh2 = [Rh, torch.empty(R.shape, dtype=torch.float32).pin_memory()]
            ev_in = [torch.cuda.Event(), torch.cuda.Event()]
            ev_sh = [torch.cuda.Event(), torch.cuda.Event()]
            ev_rl = [torch.cuda.Event(), torch.cuda.Event()]
            ev_out = [torch.cuda.Event(), torch.cuda.Event()]
            e2e_state = {"next": None, "n": 0}

            def e2e_enqueue_front(i):
                b = i & 1
                with torch.cuda.stream(cs):
                    if e2e_state["n"] >= 2:
                        cs.wait_event(ev_sh[b])               # the shift that read lbuf[b] is done
                    lbuf[b].copy_(light_h, non_blocking=True)
                    ev_in[b].record(cs)
                sstream.wait_event(ev_in[b])
                sstream.wait_event(ev_rl[b])                  # the relight that read shifted2[b] is done
                s_ = np.broadcast_to(frames[i % len(frames)][None, None, :], (1, F, 2))
                hs.haar_shift_coeffs(lbuf[b], s_, 2, out=shifted2[b], workspace=ws2[b], stream=sstream)
                ev_sh[b].record(sstream)
                e2e_state["next"] = i
                e2e_state["n"] += 1

            def e2e_step(i):   # noqa: F811 -- the c3 form
                b = i & 1
                if e2e_state["next"] != i:
                    e2e_enqueue_front(i)
                stream.wait_event(ev_sh[b])
                if i >= 2:
                    stream.wait_event(ev_out[b])              # rbuf[b]'s previous D2H is done
                hs.relight_vertices(T, shifted2[b], F, kf, out=rbuf[b])
                ev_rl[b].record(stream)
                e2e_enqueue_front(i + 1)
                ds.wait_event(ev_rl[b])
                with torch.cuda.stream(ds):
                    rh2[b].copy_(rbuf[b], non_blocking=True)
                    ev_out[b].record(ds)

        for i in range(max(1, args.warmup)):
            e2e_step(i)
        torch.cuda.synchronize()
        e2e_ev = []
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(args.steps):
            timed(e2e_step, i, e2e_ev)
        if cfg.name == "c3":
            stream.wait_event(ev_out[(args.steps - 1) & 1])   # the last radiance is on the host
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        if flush is not None:
            e_ms = sum(a_.elapsed_time(b_) for a_, b_ in e2e_ev) / len(e2e_ev)
        e2e = {"value": V / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(light_np.nbytes),
               "d2h_bytes_per_step": int(R.numel() * 4)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": V / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "faces": F, "N": N, "vertices": V, "k_face": kf,
                       "l2": "flushed (256 MB write) before every step, outside the step's timed events"
                       if flush is not None else
                       f"no flush: transfer {V * K * 4 / 1e9:.2f} GB streamed per step"},
            "roofline": {"bound": "hbm", "kernel": kernel_name, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": dom_ms, "share_of_step": dom_ms / ms},
            "gpu_launches": timed_launches, "clocks": clk.summary(), "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            t0 = time.perf_counter()
            if cfg.name == "c4":
                sub = 8
                Th = synth.transfer_rows(cfg.seed, 0, sub, F, kf)
                orelight.relight_shifted(Th, light_np[0], synth.c4_vertex_shifts(cfg.seed, V, n)[:sub].astype(float))
                full = (time.perf_counter() - t0) * V / sub
                desc = f"oracle fp64 relight_shifted on {sub}/{V} vertices (6 faces inverse-shift-forward-dot each)"
            else:
                s = np.broadcast_to(np.array([[[0.0, 17 * N / 360.0]]]), (1, F, 2))
                Lp = oshift.shift_coeffs(light_np, s, 2)
                sub = min(V, 2000)
                Th = synth.transfer_rows(cfg.seed, 0, sub, F, kf)
                t1 = time.perf_counter()
                orelight.relight(Th, Lp, F, kf)
                full = (t1 - t0) + (time.perf_counter() - t1) * V / sub
                desc = f"oracle fp64: shift of one frame + relight of {sub}/{V} rows, extrapolated"
            line["cpu_baseline"] = {"value": V / full, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                                    "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_sparse(args, cfg):
    """c5s (row f2): shift 64 frames x 6 faces of 256^2 (full pyramids), then relight 1M vertices
    whose transfer keeps K_s = 256 full-resolution coefficients (gather).  One GPU."""
    import torch

    import paper_1705_07272_b200 as hs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    V = args.vertices or cfg.vertices
    n, F, B = cfg.log2n, cfg.faces, cfg.frames
    ks, dl = cfg.extra["k_sparse"], cfg.extra["dense_levels"]
    N = 1 << n
    C = F * N * N
    idx = torch.empty((V, ks), dtype=torch.int32, device=dev)
    val = torch.empty((V, ks), dtype=torch.float32, device=dev)
    hs.hs_fill_sparse_transfer(idx, val, 0, F, n, dl, cfg.seed)
    light_np = synth.light_pyramids(cfg.seed, B, F, n)
    light = torch.from_numpy(light_np).to(dev)
    shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
    shifted = torch.empty_like(light)
    ws = torch.empty(hs.haar_shift_workspace_bytes(2, n, F, B), dtype=torch.uint8, device=dev)
    rws = torch.empty(hs.relight_sparse_workspace_bytes(C, B), dtype=torch.uint8, device=dev)
    R = torch.empty((V, B), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    dom, launches = [], {"n": 0}

    def step():
        hs.haar_shift_coeffs(light, shifts, 2, out=shifted, workspace=ws)
        launches["n"] += hs.last_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hs.relight_vertices_sparse(idx, val, shifted, out=R, workspace=rws)
        e1.record(stream)
        dom.append((e0, e1))
        launches["n"] += hs.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dom.clear()
    launches["n"] = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    dom_ms = sum(a.elapsed_time(b) for a, b in dom) / len(dom)
    peak, peak_src = hbm_peak()
    hbm_bytes = V * ks * 8 + V * B * 4 + 2 * C * B * 4
    line = {
        "metric": METRIC, "value": V / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "faces": F, "N": N, "frames": B, "vertices": V,
                   "k_sparse": ks, "l2": "sparse transfer 2 GB streamed per step; the 100 MB transposed light is "
                   "L2-resident by design (gathers)"},
        "roofline": {"bound": "hbm", "kernel": "relight_vertices_sparse (transpose + gather)",
                     "achieved": hbm_bytes / (dom_ms * 1e-3) / 1e9, "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": hbm_bytes / (dom_ms * 1e-3) / 1e9 / peak, "traffic": None,
                     "alg_bytes_per_launch": hbm_bytes, "avg_launch_ms": dom_ms, "share_of_step": dom_ms / ms,
                     "l2_gather_gbs": V * ks * B * 4 / (dom_ms * 1e-3) / 1e9,
                     "note": "bound by L2 gathers (K_s x 64 frames x 4 B per vertex), not HBM"},
        "gpu_launches": launches["n"], "clocks": clk.summary(), "e2e": None,
    }
    if not args.no_e2e:
        # end to end through the host pipeline: pinned host light in, pinned host radiance out,
        # every step; the radiance D2H runs chunk by chunk under the next chunk's relight
        from paper_1705_07272_b200.pipeline import ShiftSparseRelightPipeline
        del R
        pipe = ShiftSparseRelightPipeline(idx, val, F, n, B, chunks=4)
        light_h = torch.from_numpy(light_np).pin_memory()
        Rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        for _ in range(max(1, args.warmup)):
            pipe.step(light_h, shifts, Rh)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            done = pipe.step(light_h, shifts, Rh)
        stream.wait_event(done)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        line["e2e"] = {"value": V / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(light_np.nbytes),
                       "d2h_bytes_per_step": int(V * B * 4), "path": "pipeline.ShiftSparseRelightPipeline"}
    if not args.no_cpu_baseline:
        from oracle import relight as orelight
        from oracle import shift as oshift
        rows = 400000   # a few seconds of oracle work
        t0 = time.perf_counter()
        sh1 = oshift.shift_coeffs(light_np[:1], shifts[:1], 2)
        t_shift = time.perf_counter() - t0
        i_s, v_s = synth.sparse_transfer_rows(cfg.seed, 0, rows, F, n, ks, dl)
        Lb = np.broadcast_to(sh1.reshape(1, -1), (B, C))
        t0 = time.perf_counter()
        orelight.relight_sparse(i_s, v_s, Lb)
        t_rel = time.perf_counter() - t0
        full = t_shift * B + t_rel * (V / rows)
        line["cpu_baseline"] = {"value": V / full, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                                "sample": f"oracle fp64: shift of 1/{B} frames ({t_shift:.3f}s) + sparse relight of "
                                          f"{rows}/{V} vertices x {B} frames ({t_rel:.3f}s), extrapolated linearly"}
    print(json.dumps(line), flush=True)
    return 0


def fill_shading(hs, out, r0, faces, kf, seed, stream):
    """device twin of synth.shading_rows: hs_fill_transfer, then the same two fp32 operations"""
    hs.hs_fill_transfer(out, r0, faces, kf, seed, stream)
    sc = out[:, ::kf] * 0.5 + 0.5
    out.mul_(0.25)
    out[:, ::kf] = sc


def run_triple(args, cfg):
    """c5t (row f3): shift 64 frames x 6 faces of 256^2 to the k = 5 band, then the triple product
    of 1M vertices with separate BRDF and visibility (6 x 1024 coefficients each, qtree layout).
    One GPU."""
    import torch

    import paper_1705_07272_b200 as hs
    from paper_1705_07272_b200.pipeline import ShiftTripleRelightPipeline

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    V = args.vertices or cfg.vertices
    n, F, B, kf, k = cfg.log2n, cfg.faces, cfg.frames, cfg.k_face, cfg.band_levels
    N = 1 << n
    K = F * kf
    rq = torch.empty((V, K), dtype=torch.float32, device=dev)
    vq = torch.empty((V, K), dtype=torch.float32, device=dev)
    chunk = min(V, 65536)
    tmp = torch.empty((chunk, K), dtype=torch.float32, device=dev)
    for r0 in range(0, V, chunk):
        rows = min(chunk, V - r0)
        for dst, stream_id in ((rq, synth.STREAM_BRDF), (vq, synth.STREAM_VIS)):
            fill_shading(hs, tmp[:rows], r0, F, kf, cfg.seed, stream_id)
            hs.haar_pack_qtree(tmp[:rows].view(rows, F, kf), k, out=dst[r0:r0 + rows])
    del tmp
    light_np = synth.light_pyramids(cfg.seed, B, F, n)
    light = torch.from_numpy(light_np).to(dev)
    shifts = np.broadcast_to(synth.c5_shifts(cfg.seed, B, n)[:, None, :], (B, F, 2)).copy()
    band = torch.empty((B, F, kf), dtype=torch.float32, device=dev)
    ws = torch.empty(hs.haar_shift_workspace_bytes(2, n, F, B), dtype=torch.uint8, device=dev)
    tws_raw = torch.empty(hs.relight_triple_workspace_bytes(V, F, kf, B) + 1024, dtype=torch.uint8, device=dev)
    tws = tws_raw[(-tws_raw.data_ptr()) % 1024:]
    R = torch.empty((V, B), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    dom, launches = [], {"n": 0}

    def step():
        hs.haar_shift_coeffs(light, shifts, 2, k, out=band, workspace=ws)
        launches["n"] += hs.last_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hs.relight_vertices_triple(rq, vq, band, F, kf, out=R, workspace=tws)
        e1.record(stream)
        dom.append((e0, e1))
        launches["n"] += hs.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dom.clear()
    launches["n"] = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    dom_ms = sum(a.elapsed_time(b) for a, b in dom) / len(dom)
    peak, peak_src = hbm_peak()
    hbm_bytes = V * (2 * K * 4 + B * 4) + B * K * 4
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"{cfg.name}:triple_b{B}") if V == cfg.vertices else None
    except Exception:
        pass

    e2e = None
    if not args.no_e2e:
        light_h = torch.from_numpy(light_np).pin_memory()
        Rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        pipe = ShiftTripleRelightPipeline(rq, vq, F, n, B, k, chunks=args.e2e_chunks)
        for _ in range(max(1, args.warmup)):
            pipe.step(light_h, shifts, Rh)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            ev = pipe.step(light_h, shifts, Rh)
        stream.wait_event(ev)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        e2e = {"value": V / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(light_np.nbytes),
               "d2h_bytes_per_step": int(V * B * 4), "ms_per_step": e_ms,
               "note": "ShiftTripleRelightPipeline.step: pinned H2D of the 64 light pyramids, shift to the band, "
                       f"chunked triple product ({args.e2e_chunks} chunks), each chunk's radiance D2H overlapped; "
                       "BRDF and visibility are scene data resident in HBM"}

    line = {
        "metric": METRIC, "value": V / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "faces": F, "N": N, "frames": B, "vertices": V,
                   "k_face": kf, "l2": "no flush: BRDF + visibility (49 GB) streamed every step, far above L2"},
        "roofline": {"bound": "hbm", "kernel": "relight_vertices_triple (pack light + tile prep + tcgen05 kernel)",
                     "achieved": hbm_bytes / (dom_ms * 1e-3) / 1e9, "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": hbm_bytes / (dom_ms * 1e-3) / 1e9 / peak, "traffic": traffic,
                     "alg_bytes_per_launch": hbm_bytes, "avg_launch_ms": dom_ms, "share_of_step": dom_ms / ms},
        "gpu_launches": launches["n"], "clocks": clk.summary(), "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        t_s, rows_s, desc = oracle_sample(cfg, 256)
        line["cpu_baseline"] = {"value": rows_s / t_s, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                                "sample": desc}
    print(json.dumps(line), flush=True)
    return 0


def run_rotate(args, cfg):
    """c6r (row f1): rotate `frames` lat-long maps of 2^n x 2^n, each by its own (alpha, beta), in the
    Haar domain.  Metric: rotated maps per second; parity against the chain-rule oracle and PSNR
    against the spatial rotation on a sample."""
    import torch

    import paper_1705_07272_b200 as hs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n, B = cfg.log2n, cfg.frames
    N = 1 << n
    maps_np = synth.smooth_sphere_maps(cfg.seed, B, n)
    ang = synth.rotation_angles(cfg.seed, B)
    x = torch.from_numpy(maps_np).to(dev)
    y = torch.empty_like(x)
    ws = torch.empty(hs.haar_rotate_workspace_bytes(n, B), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    launches = {"n": 0}

    def step():
        hs.haar_rotate_coeffs(x, ang, out=y, workspace=ws)
        launches["n"] += hs.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches["n"] = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    peak, peak_src = hbm_peak()
    NN = N * N
    # algorithmic HBM bytes: read the pyramid and write the result, 4 B per coefficient each
    alg = B * NN * 4 * 2
    line = {
        "metric": "rotated_maps_per_sec", "value": B / (ms * 1e-3), "unit": "maps/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "N": N, "maps": B, "l2": "inputs 67 MB < L2; no flush"},
        "rotated_coeffs_per_sec": B * NN / (ms * 1e-3),
        "roofline": {"bound": "alu", "kernel": "haar_rotate_coeffs (all launches)",
                     "achieved": B * NN * ROT_FP64_FLOPS_PER_PIXEL / (ms * 1e-3) / 1e12, "peak": fp64_peak_tflops()[0],
                     "peak_source": fp64_peak_tflops()[1], "unit": "TFLOP/s",
                     "frac": B * NN * ROT_FP64_FLOPS_PER_PIXEL / (ms * 1e-3) / 1e12 / fp64_peak_tflops()[0],
                     "traffic": None, "alg_flops_per_launch": B * NN * ROT_FP64_FLOPS_PER_PIXEL,
                     "avg_launch_ms": ms, "share_of_step": 1.0,
                     "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak, "alg_bytes_per_launch": alg,
                     "note": "fp64 operations of the method (chain rule + bottom-up) against the fp64 FMA peak; the "
                             "chain-rule kernel is issue / latency bound (trigonometry, bilinear samples), the fp64 "
                             "pipe ~25-35 % busy"},
        "gpu_launches": launches["n"], "clocks": clk.summary(), "e2e": None,
    }
    if not args.no_e2e:
        # host buffers through pipeline.RotatePipeline: chunked, copies under the rotation
        from paper_1705_07272_b200.pipeline import RotatePipeline
        pipe = RotatePipeline(B, n, dev, chunks=4)
        x_h = torch.from_numpy(maps_np).pin_memory()
        y_h = torch.empty((B, NN), dtype=torch.float32).pin_memory()
        for _ in range(max(1, args.warmup)):
            pipe.step(x_h, ang, y_h)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            done = pipe.step(x_h, ang, y_h)
        stream.wait_event(done)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        line["e2e"] = {"value": B / (e_ms * 1e-3), "unit": "maps/s", "h2d_bytes_per_step": int(maps_np.nbytes),
                       "d2h_bytes_per_step": int(B * NN * 4), "path": "pipeline.RotatePipeline"}
    if not args.no_cpu_baseline:
        from oracle import rotate as orot
        yh = y.cpu().numpy()
        k = 1024   # a few seconds of oracle work
        t0 = time.perf_counter()
        refs = [orot.rotate_coeffs_chain(maps_np[b], *ang[b]) for b in range(k)]   # the parity oracle
        dt = time.perf_counter() - t0
        errs = [float(np.linalg.norm(yh[b] - refs[b]) / np.linalg.norm(refs[b])) for b in range(k)]
        line["parity_vs_oracle"] = {"max_rel_l2": max(errs), "maps": k, "tol": 1e-5}
        ps = [orot.psnr(yh[b], orot.rotate_coeffs(maps_np[b], *ang[b])) for b in range(16)]
        line["psnr_vs_spatial_db"] = {"min": min(ps), "median": float(np.median(ps)), "maps": 16}
        line["cpu_baseline"] = {"value": k / dt, "unit": "maps/s", "cores": cpu_threads(), "kind": "oracle",
                                "sample": f"oracle fp64 chain-rule rotation of {k}/{B} maps ({dt:.3f}s)"}
    print(json.dumps(line), flush=True)
    return 0


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_ranks(args) -> None:
    """`--gpus N` is the number of ranks, one per GPU.  Under torchrun WORLD_SIZE must equal N;
    without it (a plain `python bench.py --gpus N`) the script re-executes itself under
    torch.distributed.run with N local ranks (rendezvous on 127.0.0.1) and exits with its status."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank per GPU",
                  file=sys.stderr)
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    if args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"[bench] --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}", file=sys.stderr)
            sys.exit(2)
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def run_shade(args, cfg):
    """c7s (rows f1 + f3, the paper's shading): shift 64 light frames (lat-long
    N x N) to the band, then relight_vertices_brdf_rotated -- one BRDF rotated per vertex normal in
    the Haar domain, triple product with the vertex's visibility.  One GPU."""
    import torch

    import paper_1705_07272_b200 as hs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    V = args.vertices or cfg.vertices
    n, B, k, kf = cfg.log2n, cfg.frames, cfg.band_levels, cfg.k_face
    N = 1 << n
    brdf = torch.from_numpy(synth.smooth_sphere_maps(cfg.seed, 1, n)[0]).to(dev)
    vis_np = synth.shading_rows(cfg.seed, 0, V, 1, kf, synth.STREAM_VIS)
    vq = hs.haar_pack_qtree(torch.from_numpy(vis_np).to(dev).view(V, 1, kf), k).view(V, kf)
    rng = np.random.default_rng([cfg.seed, 7])
    nv = rng.normal(size=(V, 3))
    nv /= np.linalg.norm(nv, axis=1, keepdims=True)
    normals = np.stack([np.arccos(np.clip(nv[:, 1], -1.0, 1.0)), np.mod(np.arctan2(nv[:, 0], nv[:, 2]), 2 * np.pi)], 1)
    light_np = synth.light_pyramids(cfg.seed, B, 1, n)
    light = torch.from_numpy(light_np).to(dev)
    shifts = np.stack([np.zeros(B), np.arange(B) * N / 64.0], axis=1)[:, None, :]   # azimuth steps (global shift)
    band = torch.empty((B, 1, kf), dtype=torch.float32, device=dev)
    sws = torch.empty(hs.haar_shift_workspace_bytes(2, n, 1, B), dtype=torch.uint8, device=dev)
    need = hs.relight_brdf_rotated_workspace_bytes(n, k, B)
    wraw = torch.empty(need + 1024, dtype=torch.uint8, device=dev)
    ws = wraw[(-wraw.data_ptr()) % 1024:]
    R = torch.empty((V, B), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    launches = {"n": 0}

    def step():
        hs.haar_shift_coeffs(light, shifts, 2, k, out=band, workspace=sws)
        launches["n"] += hs.last_launch_count()
        hs.relight_vertices_brdf_rotated(brdf, normals, vq, band.view(B, kf), k, out=R, workspace=ws)
        launches["n"] += hs.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches["n"] = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        time.sleep(0.01)
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    peak, peak_src = hbm_peak()
    NN = N * N
    # algorithmic HBM bytes of the composed call: the rotated BRDF pyramids written and read back
    # (4 B x N^2 each way), the qtree bands (4 B x kf each way), visibility 4 B x kf, radiance 4 B x B
    alg = V * (NN * 8 + kf * 12 + B * 4) + B * kf * 4
    e2e = None
    if not args.no_e2e:
        light_h = torch.from_numpy(light_np).pin_memory()
        Rh = torch.empty((V, B), dtype=torch.float32).pin_memory()
        for _ in range(max(1, args.warmup)):
            light.copy_(light_h, non_blocking=True)
            step()
            Rh.copy_(R, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            light.copy_(light_h, non_blocking=True)
            step()
            Rh.copy_(R, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        e2e = {"value": V / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(light_np.nbytes),
               "d2h_bytes_per_step": int(V * B * 4), "ms_per_step": e_ms,
               "note": "pinned H2D of the 64 light pyramids, shift, composed rotate + triple call, pinned D2H of R; "
                       "BRDF, normals and visibility are scene data"}
    line = {
        "metric": METRIC, "value": V / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "faces": 1, "N": N, "frames": B, "vertices": V,
                   "k_face": kf, "l2": "no flush"},
        "roofline": {"bound": "alu", "kernel": "relight_vertices_brdf_rotated (rotation + pack + triple product)",
                     "achieved": V * N * N * ROT_FP64_FLOPS_PER_PIXEL / (ms * 1e-3) / 1e12,
                     "peak": fp64_peak_tflops()[0], "peak_source": fp64_peak_tflops()[1], "unit": "TFLOP/s",
                     "frac": V * N * N * ROT_FP64_FLOPS_PER_PIXEL / (ms * 1e-3) / 1e12 / fp64_peak_tflops()[0],
                     "traffic": None, "alg_flops_per_launch": V * N * N * ROT_FP64_FLOPS_PER_PIXEL,
                     "avg_launch_ms": ms, "share_of_step": 1.0,
                     "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak, "alg_bytes_per_launch": alg,
                     "note": "the per-vertex BRDF rotation's fp64 operations (as c6r) against the fp64 FMA peak; the "
                             "triple product and the pack are a few % of the call"},
        "gpu_launches": launches["n"], "clocks": clk.summary(), "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        from oracle import relight as orelight
        from oracle import rotate as orot
        rows = 24
        t0 = time.perf_counter()
        band_np = np.stack([synth_shift_band(light_np[b, 0], shifts[b, 0], k) for b in range(B)])
        rho = np.stack([orot.rotate_coeffs_chain(synth.smooth_sphere_maps(cfg.seed, 1, n)[0].astype(np.float64),
                                                 float(normals[v, 0]), float(normals[v, 1]))[:kf]
                        for v in range(rows)])
        orelight.relight_triple(rho, vis_np[:rows].astype(np.float64), band_np[:, None, :], 1, kf)
        t_s = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": rows / t_s, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                                "sample": f"oracle fp64 on {rows} of {V} vertices (measured): the 64 frames' shift, "
                                          f"{rows} chain-rule rotations of the BRDF, the triple integral"}
    print(json.dumps(line), flush=True)
    return 0


def synth_shift_band(pyr, shift2, k):
    """oracle shift of one lat-long pyramid, band prefix (CPU baseline of c7s)"""
    from oracle import shift as oshift
    return oshift.shift_coeffs(pyr[None, None, :].astype(np.float64), np.asarray(shift2)[None, None, :], 2)[0, 0, :4 ** k]


def main():
    args = parse_args()
    launch_ranks(args)
    cfg = synth.config(args.config)
    if args.vertices:
        cfg = synth.Config(**{**cfg.__dict__, "vertices": args.vertices})
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.name in ("c2", "c3", "c4"):
        return run_aux(args, cfg)
    if cfg.name == "c5s":
        return run_sparse(args, cfg)
    if cfg.name == "c5t":
        return run_triple(args, cfg)
    if cfg.name == "c6r":
        return run_rotate(args, cfg)
    if cfg.name == "c7s":
        return run_shade(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
