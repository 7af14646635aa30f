#!/usr/bin/env python
"""bench.py — B200 video front end: motion -> CCL -> blob stats -> tracking.

Metric (BASELINE.json): frames/sec (1080p, device-timed) motion+segment+track
and the fraction of the HBM roofline.  Workload: S
independent 1920x1080 grayscale camera streams per GPU, each a C3-recipe
clip (20 moving blobs with occlusions/merges, stream s uses shape seed
mix_seed(3, s)); a step advances every stream by one frame through the full
path (Mean background W=91 update + threshold, 8-connected CCL with
min_area 4 and canonical relabel, per-blob area/bbox/centroid, mean-shift
tracking with spawn/retire/log).  The W-1 = 90 window-fill frames run before
timing (they emit no mask).  Inputs are synthetic (device-rasterised from
the reference generator's integer rectangles, never inside a timed region).
Every step touches > 126 MB (ring slots alone are S x 2 MB read + written),
so consecutive steps do not hit L2.

Multi-GPU: streams are independent, so ranks shard them (rank r owns
streams r*S .. r*S+S-1) with no data-path collective — weak scaling.  The
timed region is bracketed by barrier + synchronize, the time is the MAX over
ranks (all_reduce MAX).

  python bench.py                      # N=1, defaults
  python bench.py --impl reference     # reference CPU path on host cores
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

W_DEFAULT = 91
WIDTH, HEIGHT = 1920, 1080
PX = WIDTH * HEIGHT
MOTION_BYTES_PER_PX = 8   # frame 1 + evict 1 + insert 1 + u16 sum 2+2 + mask 1
PATH_BYTES_PER_PX = 12    # + int32 labels
MORPH_BYTES_PER_PX = 2    # fused 3x3 open: mask in 1 + mask out 1 (halo re-reads are not algorithmic)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--streams", type=int, default=64, help="streams per GPU (C5: 64)")
    p.add_argument("--cpu-threads", type=int, default=0, help="reference/baseline host threads (0 = all, capped)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- reference
def host_frame(clip, t):
    from paper_1310_3322_b200.synth import raster_host
    return raster_host(clip, clip.rects(t))


def run_reference_cpu(n_streams, threads, steps, warmup, stream_base=0):
    """The unmodified reference (oracle/_ref) on host threads: fill the W=91
    window untimed, then time `steps` steps of one frame per stream."""
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from paper_1310_3322_b200.synth import recipe
    from tests import _oracle as O
    import ctypes as C
    kind = "reference" if O.ref_available() else "port"
    L = O.ref_lib() if kind == "reference" else None
    if L is None:
        raise RuntimeError("oracle/_ref/libteamrec_ref.so is not built (run make -C oracle where the reference is)")
    L.ref_streams_create.restype = C.c_void_p
    L.ref_streams_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_streams_step.restype = C.c_int64
    L.ref_streams_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.ref_streams_destroy.argtypes = [C.c_void_p]
    mc, sc, tc = MOTION_CFG(), SEG_CFG(), TRACKER_CFG()
    h = L.ref_streams_create(n_streams, WIDTH, HEIGHT, 1, C.byref(mc), C.byref(sc), C.byref(tc))
    clips = [recipe("C5", stream_base + s) for s in range(n_streams)]
    ptrs = (C.c_void_p * n_streams)()

    def step(t):
        fr = [host_frame(c, t) for c in clips]
        for i, f in enumerate(fr):
            ptrs[i] = f.ctypes.data
        t0 = time.perf_counter()
        n = L.ref_streams_step(h, ptrs, threads)
        return n, time.perf_counter() - t0

    t = 0
    for _ in range(W_DEFAULT - 1 + warmup):
        step(t)
        t += 1
    frames, secs = 0, 0.0
    for _ in range(steps):
        n, dt = step(t)
        t += 1
        frames += n
        secs += dt
    L.ref_streams_destroy(h)
    return frames / secs, frames, secs, kind


def cpu_threads(requested):
    n = os.cpu_count() or 1
    try:  # keep the reference's 205 MB/stream state within a quarter of free RAM
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
        n = min(n, max(1, int(avail_kb * 1024 * 0.25 / 230e6)))
    except Exception:
        pass
    n = min(n, 64)
    return requested if requested > 0 else n


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_main(args, rank, world):
    if rank != 0:
        return
    threads = cpu_threads(args.cpu_threads)
    fps, frames, secs, kind = run_reference_cpu(threads, threads, args.steps, args.warmup)
    sample = (f"{threads} C5 streams x {args.steps} steady frames each after a {W_DEFAULT - 1}-frame window fill "
              f"(+{args.warmup} warmup), one stream per host thread; {cpu_model()}")
    line = {
        "impl": "reference", "metric": "frames/sec (1080p, device-timed) motion+segment+track", "value": fps,
        "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C5: independent 1920x1080 C3-recipe camera streams", "streams": threads,
                   "window": W_DEFAULT, "host_threads": threads},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------ multi-rank plumbing
def shard(rank: int, streams_per_rank: int):
    """Streams owned by `rank` (weak scaling: every rank owns the same number
    of independent streams; no data-path collective)."""
    return list(range(rank * streams_per_rank, (rank + 1) * streams_per_rank))


def max_over_ranks(x: float, world: int, device="cpu") -> float:
    """The job's time is the slowest rank's (all_reduce MAX; nccl tensors on
    the rank's GPU, gloo on the host)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_fps(streams_per_rank: int, world: int, steps: int, seconds: float) -> float:
    """Whole-job frames/s: every rank advanced its streams `steps` frames."""
    return streams_per_rank * world * steps / seconds


# -------------------------------------------------------------------- ours
def make_frames(trb, clips, n_frames, stream):
    """Device-rasterised clip frames: uint8 [S, n_frames, px]."""
    import torch
    S = len(clips)
    from paper_1310_3322_b200 import api
    buf = torch.empty((S, n_frames, PX), dtype=torch.uint8, device="cuda")
    for s, c in enumerate(clips):
        rects = [c.rects(t) for t in range(n_frames)]
        api.synth_raster_frames(buf[s, 0].data_ptr(), PX, WIDTH, HEIGHT, 1, c.background, rects, c.colors(),
                                stream.cuda_stream)
    torch.cuda.synchronize()
    return buf


_HOST_AFFINITY = None  # the process's cores before bind_to_gpu_numa_node (the CPU baseline uses them all)


def bind_to_gpu_numa_node(local_rank):
    """Run this rank on the host cores local to its GPU (NVML affinity): the
    pinned staging / frame buffers are then first-touched on the GPU's NUMA
    node, so the e2e H2D copies do not cross the socket interconnect."""
    global _HOST_AFFINITY
    _HOST_AFFINITY = os.sched_getaffinity(0)
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
        pynvml.nvmlShutdown()
        return len(cpus)
    except Exception:
        return 0


def ours_main(args, rank, world, local_rank):
    bind_to_gpu_numa_node(local_rank)
    import torch
    import torch.distributed as dist
    import paper_1310_3322_b200 as trb
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from paper_1310_3322_b200.synth import recipe

    S, K, Wm = args.streams, args.steps, args.warmup
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    clips = [recipe("C5", s) for s in shard(rank, S)]
    fill = W_DEFAULT - 1
    e2e_steps = 0 if args.no_e2e else K
    n_frames = fill + Wm + K + K
    assert n_frames <= 300, "recipe clips have 300 frames"
    frames = make_frames(trb, clips, n_frames, stream)
    st = trb.Streams(S, WIDTH, HEIGHT, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), device=local_rank)
    ptrs = [[frames[s, t].data_ptr() for s in range(S)] for t in range(n_frames)]
    t = 0
    with torch.cuda.stream(stream):
        for _ in range(fill + Wm):
            st.step_device(ptrs[t], stream.cuda_stream)
            t += 1
    torch.cuda.synchronize()
    assert st.has_output

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- timed region: K steps, device-resident inputs
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    t_timed0 = t
    ev0.record(stream)
    for _ in range(K):
        st.step_device(ptrs[t], stream.cuda_stream)
        launches += st.last_launches
        t += 1
    st.join(stream.cuda_stream)  # the last step's tracking (internal stream) is inside the timed region
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
    clk = clocks.stop()

    # ---- per-stage kernel times (second pass of K steps, events per stage)
    #      and the tracker's window pixels (its algorithmic frame reads)
    from paper_1310_3322_b200 import api
    api.debug_stats(reset=True)
    st.profile(True)
    for _ in range(K):
        st.step_device(ptrs[t], stream.cuda_stream)
        t += 1
    torch.cuda.synchronize()
    stage_ms, prof_steps = st.profile_read()
    st.profile(False)
    stage_ms = stage_ms / max(1, prof_steps)
    track_px = api.debug_stats(reset=True).get("meanshift_window_px", 0) / max(1, prof_steps)

    # ---- the fused 3x3 morphology kernel (north-star kernel (2); OFF in the
    #      reference-parity workload): open (erode -> dilate, one fused pass)
    #      on this step's 64 x 1080p masks, CUDA events around K launches
    mask0, _ = st.device_planes(0)
    morph_out = torch.empty((S, PX), dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            api.morph_device(mask0, morph_out.data_ptr(), WIDTH, HEIGHT, S, 3, stream.cuda_stream)
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for _ in range(K):
            api.morph_device(mask0, morph_out.data_ptr(), WIDTH, HEIGHT, S, 3, stream.cuda_stream)
        m1.record(stream)
    torch.cuda.synchronize()
    morph_ms = m0.elapsed_time(m1) / K
    del morph_out

    # ---- e2e through the C-ABI with host buffers (pinned), H2D + D2H timed
    e2e = None
    if e2e_steps:
        # Same work as `value`: a second handle is advanced through the same
        # fill + warm-up frames, then the SAME K frames as the device-timed
        # region go through the host API.  Pinned host frames and per-step
        # pinned result rows; the pipelined API overlaps step k+1's H2D with
        # step k's kernels, every step's result (S blob counts) is read back.
        st.synchronize()
        del st
        st = trb.Streams(S, WIDTH, HEIGHT, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), device=local_rank)
        with torch.cuda.stream(stream):
            for k in range(t_timed0):
                st.step_device(ptrs[k], stream.cuda_stream)
        torch.cuda.synchronize()
        # each step's S frames back to back in one pinned buffer (as a capture
        # ring would hold them): the host path then issues one H2D copy
        host_steps = [frames[:, t_timed0 + k].cpu().contiguous().pin_memory().numpy() for k in range(e2e_steps)]
        host = [[hs[s] for s in range(S)] for hs in host_steps]
        res = torch.zeros((e2e_steps, S), dtype=torch.int32).pin_memory().numpy()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            st.step_host_async(host[k], res[k], stream.cuda_stream)
        st.synchronize()
        torch.cuda.synchronize()
        secs = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": aggregate_fps(S, world, e2e_steps, secs), "unit": "frames/s", "h2d_bytes_per_step": S * PX,
               "d2h_bytes_per_step": 4 * S,
               "frames": "the device-timed steps' frames, through trb_streams_step_host_async (second handle)"}
    st.synchronize()

    value = aggregate_fps(S, world, K, ms / 1e3)
    peak, peak_kind = measured_peaks()

    def dram_traffic(name):  # ncu dram bytes per launch, when captured for this stream count
        tp = os.path.join(ROOT, "profiles", name)
        try:
            with open(tp) as f:
                d = json.load(f)
            return d["dram_bytes_per_launch"] if d.get("streams") == S else None
        except Exception:
            return None

    motion_ms = stage_ms[0]
    achieved = MOTION_BYTES_PER_PX * S * PX / (motion_ms / 1e3) / 1e9
    roofline_motion = {"bound": "hbm", "kernel": "motion_mean_kernel", "achieved": achieved, "peak": peak,
                       "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                       "traffic": dram_traffic("motion_dram_bytes.json"),
                       "bytes_per_launch": MOTION_BYTES_PER_PX * S * PX}
    morph_achieved = MORPH_BYTES_PER_PX * S * PX / (morph_ms / 1e3) / 1e9
    roofline_morph = {"bound": "hbm", "kernel": "morph_strip_kernel<open> (erode+dilate fused)",
                      "achieved": morph_achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                      "frac": morph_achieved / peak, "traffic": None, "bytes_per_launch": MORPH_BYTES_PER_PX * S * PX,
                      "ms_per_launch": morph_ms,
                      "note": "not on the parity path (the reference has no morphology); one launch per step when "
                              "MotionConfig.morph is set; back-to-back launches on the same 133 MB of masks"}
    # the dominant kernel: track_meanshift_kernel.  SURVEY §8(d): tracking's
    # algorithmic bytes are its frame reads, window px x iterations x channels
    ms_ms = stage_ms[2]
    ms_bytes = track_px * 1
    ms_achieved = ms_bytes / (ms_ms / 1e3) / 1e9 if ms_ms > 0 else 0.0
    roofline = {"bound": "hbm", "kernel": "track_meanshift_kernel", "achieved": ms_achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": ms_achieved / peak,
                "traffic": dram_traffic("meanshift_dram_bytes.json"), "bytes_per_launch": ms_bytes,
                "note": "exact-order fp64 sums (sequential-sum reproduction) make this kernel latency/"
                        "barrier bound, not bandwidth bound: ncu IPC ~1.2 of 4, ~26% of warp-stall samples "
                        "in cluster-barrier waits, ~550 cycles per element-walk step on an idle GPU; "
                        "profiles/r01_meanshift_ncu_full.txt, DESIGN.md 3.4"}
    path_gbs = PATH_BYTES_PER_PX * S * PX / (ms / K / 1e3) / 1e9
    line = {
        "metric": "frames/sec (1080p, device-timed) motion+segment+track", "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C5: independent 1920x1080 C3-recipe camera streams (20 blobs, occlusions/merges)",
                   "streams_per_gpu": S, "streams_total": S * world, "window": W_DEFAULT, "threshold": 25,
                   "connectivity": 8, "min_area": 4, "k_clusters": 16,
                   "parallelism": f"streams sharded over {world} GPU(s), no collective",
                   "l2": f"inputs larger than L2 ({S * 4 * PX / 1e6:.0f} MB of ring traffic per step)",
                   "stage_ms_per_step": {"motion": stage_ms[0], "ccl_stats": stage_ms[1],
                                         "track_meanshift": stage_ms[2], "track_gate_spawn": stage_ms[3]},
                   "track_window_px_per_step": track_px,
                   "stage_timing": "separate pass of K steps with CUDA events between stages",
                   "path_hbm_frac": path_gbs / peak},
        "roofline": roofline, "roofline_motion": roofline_motion, "roofline_morph": roofline_morph,
        "gpu_launches": launches, "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if _HOST_AFFINITY:
            os.sched_setaffinity(0, _HOST_AFFINITY)  # the reference baseline gets every host core
        threads = cpu_threads(args.cpu_threads)
        fps, frames_done, secs, kind = run_reference_cpu(threads, threads, 2, 0)
        line["cpu_baseline"] = {
            "value": fps, "unit": "frames/s", "cores": threads, "kind": kind,
            "sample": f"{threads} C5 streams x 2 steady frames after the {W_DEFAULT - 1}-frame fill, "
                      f"one stream per thread; {cpu_model()}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_main(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        ours_main(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
