#!/usr/bin/env python
"""bench.py — B200 video front end: motion -> CCL -> blob stats -> tracking.

Metric (BASELINE.json): frames/sec (1080p, device-timed) motion+segment+track
and the fraction of the HBM roofline.  Workloads are SURVEY §8(d)'s recipes
(the reference generator's clips, synth.hpp:45-101), default C5:

  C1  320x240, 3 blobs                 one stream (BASELINE configs[0])
  C2  640x480, 8 players               one stream (configs[1]); C2M = C2 with
                                        the fused 3x3 open (extension, no parity)
  C3  1920x1080, 20 crossing blobs     one stream (configs[2])
  C4  3840x2160, 50 crossing blobs     one stream (configs[3])
  C5  64 independent C3-recipe streams per GPU (configs[4]); stream s uses
      shape seed mix_seed(3, s).  --streams-total T instead fixes T streams
      over the job (strong scaling: stream s on GPU floor(s*G/T)).

A step advances every stream of the GPU by one frame through the full path
(Mean background W=91 + threshold, 8-connected CCL with min_area 4 and
canonical relabel, per-blob area/bbox/centroid, mean-shift tracking with
spawn/retire/log).  The W-1 = 90 window-fill frames run before timing (they
emit no mask).  Inputs are device-rasterised from the reference generator's
integer rectangles (never inside a timed region); tests hash them against
the reference's own frames (tests/test_gpu_bench_parity.py).

  value   device-timed frames/s, inputs resident in HBM (CUDA events around
          K steps on the launch stream, max over ranks)
  e2e     the same through the C ABI's host path (trb_streams_step_host_async
          _out): pinned host frames -> H2D -> kernels -> D2H of every
          stream's blob table and the frame's track-log entries, wall clock
          over >= 100 steps after a host-path warm-up
  verify  track logs of a few streams after the timed region == the
          unmodified reference's on the same frames

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).  Streams are independent:
ranks shard them with no data-path collective; the timed region is
bracketed by barrier + synchronize and the time is the max over ranks.

  python bench.py                        # C5, N=1
  python bench.py --config all           # one line per config (C1..C5, C2M)
  python bench.py --gpus 8 --streams-total 64
  python bench.py --impl reference       # the reference CPU path (64 C5 streams, all host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_DEFAULT = 91
HBM_NOMINAL_GBS = 8000.0  # B200 nominal HBM3e (also report against it)
METRIC = "frames/sec (1080p, device-timed) motion+segment+track"
MOTION_BYTES_PER_PX = 8   # frame 1 + evict 1 + insert 1 + u16 sum 2+2 + mask 1
PATH_BYTES_PER_PX = 12    # + int32 labels
MORPH_BYTES_PER_PX = 2    # fused 3x3 open: mask in 1 + mask out 1 (halo re-reads are not algorithmic)
# incremental Mode, the common push (evicted and new sample in one bin): frame 1 + ring evict/insert 2 +
# bin sum read/write 4 + mode bin read/write 2 + its count 1 + mask 1 + 1 (the mode bin's sum when it
# differs); a bin change adds the two counters (4 B), a rescan 1 B per bin (not counted)
MODE_BYTES_PER_PX = 12
CLIP_FRAMES = 300         # the recipes' clip length (n_frames is part of the recipe)

CONFIGS = {
    "C1": dict(recipe="C1", streams=1, desc="C1: one 320x240 clip, 3 moving blobs (BASELINE configs[0])"),
    "C2": dict(recipe="C2", streams=1, desc="C2: one 640x480 UC-Teamwork-like clip, 8 players (configs[1])"),
    "C2M": dict(recipe="C2", streams=1, morph=3,
                desc="C2 + fused 3x3 open (erode+dilate) inside the step (extension: no reference parity)"),
    "C3": dict(recipe="C3", streams=1, desc="C3: one 1920x1080 clip, 20 crossing blobs with occlusions/merges "
                                            "(configs[2])"),
    "C4": dict(recipe="C4", streams=1, desc="C4: one 3840x2160 clip, 50 crossing blobs (configs[3])"),
    "C5": dict(recipe="C5", streams=64, desc="C5: independent 1920x1080 C3-recipe camera streams (20 blobs, "
                                              "occlusions/merges), 64 per GPU (configs[4])"),
    "C5MODE": dict(recipe="C5", streams=64, method=1,
                   desc="C5 with the Mode background (MotionConfig.method = mode, 32 bins; SURVEY 8(f) row 1)"),
}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C5", help="C1|C2|C2M|C3|C4|C5|all")
    p.add_argument("--streams", type=int, default=0, help="streams per GPU (default: the config's; C5 64)")
    p.add_argument("--streams-total", type=int, default=0,
                   help="strong scaling: this many streams over the whole job (stream s on GPU floor(s*G/T))")
    p.add_argument("--e2e-steps", type=int, default=100)
    p.add_argument("--verify-streams", type=int, default=2, help="streams whose logs are checked (0 = off)")
    p.add_argument("--cpu-threads", type=int, default=0, help="reference arm host threads (0 = nproc)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dry-run", action="store_true", help="plumbing only (no kernels): rank/shard report")
    return p.parse_args(argv)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # the sampler is up before the timed region starts
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self, t0=None, t1=None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        window = [ln for ts, ln in self.lines if t0 is None or (t0 - 0.06 <= ts <= t1 + 0.06)]
        lines = window if window else [ln for _, ln in self.lines]
        for ln in lines:
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
                "samples": len(sm), "samples_in_timed_region": len(window)}


# ------------------------------------------------------------- host facts
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            return next(int(l.split()[1]) for l in f if l.startswith("MemAvailable")) / 1e6
    except Exception:
        return None


_HOST_AFFINITY = None  # the process's cores before bind_to_gpu_numa_node (the CPU baseline uses them all)


def bind_to_gpu_numa_node(local_rank):
    """Run this rank on the host cores local to its GPU (NVML affinity): the
    pinned staging / frame buffers are then first-touched on the GPU's NUMA
    node, so the e2e H2D copies do not cross the socket interconnect.
    Returns what happened (reported in the JSON line)."""
    global _HOST_AFFINITY
    _HOST_AFFINITY = os.sched_getaffinity(0)
    info = {"nproc": os.cpu_count(), "affinity_before": len(_HOST_AFFINITY), "pynvml": False, "bound_cpus": None,
            "numa_node": None}
    try:
        import pynvml
        info["pynvml"] = True
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= _HOST_AFFINITY
        if cpus:
            os.sched_setaffinity(0, cpus)
            info["bound_cpus"] = len(cpus)
        try:
            bus = pynvml.nvmlDeviceGetPciInfo(h).busId
            bus = (bus.decode() if isinstance(bus, bytes) else bus).lower()[4:]  # 00000000:1b:00.0 -> 0000:1b:00.0
            with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
                info["numa_node"] = int(f.read())
        except Exception:
            pass
        pynvml.nvmlShutdown()
    except Exception as e:  # noqa: BLE001
        info["bind_error"] = f"{type(e).__name__}: {e}"
        print(f"[bench] warning: NUMA binding skipped ({info['bind_error']})", file=sys.stderr)
    return info


# ------------------------------------------------------ multi-rank plumbing
def shard(rank: int, world: int, streams_per_rank: int, streams_total: int = 0):
    """Streams owned by `rank`.  Weak scaling (streams_total 0): every rank
    owns streams_per_rank independent streams, rank r the block starting at
    r*streams_per_rank.  Strong scaling: streams_total streams over the job,
    stream s on rank floor(s*world/streams_total)."""
    if streams_total:
        return [s for s in range(streams_total) if s * world // streams_total == rank]
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


def sum_over_ranks(x: float, world: int, device="cpu") -> float:
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def aggregate_fps(frames_all_ranks: float, seconds: float) -> float:
    """Whole-job frames/s: frames every rank advanced over the job's time."""
    return frames_all_ranks / seconds


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(argv, n):
    """`--gpus N` run directly: start N ranks of this script (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


# ------------------------------------------------------------- reference
def ref_lib():
    from tests import _oracle as O
    import ctypes as C
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/libteamrec_ref.so is not built (run make -C oracle where the reference is)")
    L = O.ref_lib()
    L.ref_streams_create.restype = C.c_void_p
    L.ref_streams_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_streams_step.restype = C.c_int64
    L.ref_streams_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.ref_streams_destroy.argtypes = [C.c_void_p]
    return L


def run_reference_streams(clips, threads, steps, warmup, mcfg=None):
    """The unmodified reference (oracle/_ref) per-frame loop
    (MotionDetector::push -> label_blocked(sequential) -> Tracker::process)
    for every clip, streams spread over `threads` host threads: fill the
    window untimed, then time `steps` steps of one frame per stream.
    Returns (frames/s, frames, seconds)."""
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from paper_1310_3322_b200.synth import raster_host
    import ctypes as C
    L = ref_lib()
    mc, sc, tc = mcfg or MOTION_CFG(), SEG_CFG(), TRACKER_CFG()
    c0 = clips[0]
    n = len(clips)
    h = L.ref_streams_create(n, c0.width, c0.height, c0.channels, C.byref(mc), C.byref(sc), C.byref(tc))
    ptrs = (C.c_void_p * n)()

    def step(t):
        fr = [raster_host(c, c.rects(t)) for c in clips]
        for i, f in enumerate(fr):
            ptrs[i] = f.ctypes.data
        t0 = time.perf_counter()
        k = L.ref_streams_step(h, ptrs, threads)
        return k, time.perf_counter() - t0

    t = 0
    for _ in range(mc.window - 1 + warmup):
        step(t)
        t += 1
    frames, secs = 0, 0.0
    for _ in range(steps):
        k, dt = step(t)
        t += 1
        frames += k
        secs += dt
    L.ref_streams_destroy(h)
    return frames / secs, frames, secs


def reference_single_thread(clip, steady, mcfg=None):
    """the reference on ONE thread, steady fps of one clip
    and its motion / segmentation / tracking split (ref_run_streams' per-stage
    steady_clock timers), over the window fill plus `steady` frames."""
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from tests import _oracle as O
    import ctypes as C
    L = ref_lib()
    mc = mcfg or MOTION_CFG()
    n = min(CLIP_FRAMES, mc.window - 1 + steady)
    frames, _ = O.ref_frames(clip, n)
    ptrs = (C.c_void_p * 1)(frames.ctypes.data)
    steady_out = np.zeros(1, np.int64)
    stage = np.zeros(3)
    wall = C.c_double(0)
    rc = L.ref_run_streams(1, 1, clip.width, clip.height, clip.channels, ptrs, n, C.byref(mc), C.byref(SEG_CFG()),
                           C.byref(TRACKER_CFG()), steady_out.ctypes.data, C.byref(wall), None, stage.ctypes.data)
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    k = int(steady_out[0])
    busy = float(stage.sum())
    return {"value": k / busy, "unit": "frames/s", "cores": 1, "kind": "reference",
            "sample": f"one {clip.width}x{clip.height} stream, {mc.window - 1} fill + {k} steady frames, one thread "
                      f"(ref_run_streams per-stage steady_clock); {cpu_model()}",
            "split_ms_per_frame": {"motion": 1e3 * stage[0] / k, "segmentation": 1e3 * stage[1] / k,
                                   "tracking": 1e3 * stage[2] / k}}


CPU_STEADY = {"C1": 200, "C2": 150, "C2M": 150, "C3": 40, "C4": 12, "C5": 40, "C5MODE": 10}


def reference_main(args, rank, world):
    """--impl reference: the reference's own CPU path for the same config on
    the box's host cores (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    from paper_1310_3322_b200.synth import recipe
    name = "C5" if args.config == "all" else args.config
    cfg = CONFIGS[name]
    threads = args.cpu_threads or os.cpu_count() or 1
    # the job's streams (weak: per-GPU streams x world), capped at 64: the CPU
    # path's throughput is set by its threads once streams >= threads, and
    # 64 reference streams already hold ~13 GB of host state
    S_job = args.streams_total or (args.streams or cfg["streams"]) * world
    S = min(S_job, 64)
    clips = [recipe(cfg["recipe"], s) for s in range(S)] if cfg["recipe"] == "C5" else [recipe(cfg["recipe"])] * S
    fps, frames, secs = run_reference_streams(clips, threads, args.steps, args.warmup)
    sample = (f"{S} {name} stream(s) x {args.steps} steady frames each after a {W_DEFAULT - 1}-frame window fill "
              f"(+{args.warmup} warm-up), {threads} host threads, one stream per thread at a time; {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.streams_total else "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": cfg["desc"], "name": name, "streams_total": S_job, "streams_run_on_cpu": S,
                   "window": W_DEFAULT, "host_threads": threads, "nproc": os.cpu_count()},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def verify_logs(clips, logs, n_frames, mcfg=None):
    """The unmodified reference over the same frames: track logs equal."""
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from tests import _oracle as O
    fr = [O.ref_frames(c, n_frames)[0] for c in clips]
    c0 = clips[0]
    ref = O.ref_run_streams_detail(fr, c0.width, c0.height, c0.channels, mcfg or MOTION_CFG(), SEG_CFG(), TRACKER_CFG(),
                                   len(clips), bcap=1, lcap=1 << 16)
    return [r["log"].tobytes() == lg.tobytes() for r, lg in zip(ref, logs)], [len(lg) for lg in logs]


def ours_config(args, name, rank, world, local_rank, bind_info, first):
    import torch
    import torch.distributed as dist
    import paper_1310_3322_b200 as trb
    from paper_1310_3322_b200 import api
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from paper_1310_3322_b200.synth import device_frames, recipe

    cfg = CONFIGS[name]
    dev = torch.device("cuda", local_rank)
    per_rank = args.streams or cfg["streams"]
    mine = shard(rank, world, per_rank, args.streams_total)
    if cfg["recipe"] == "C5":
        clips = [recipe("C5", s) for s in mine]
    else:
        clips = [recipe(cfg["recipe"]) for _ in mine]
    S = len(clips)
    assert S >= 1, "every rank needs at least one stream"
    c0 = clips[0]
    px = c0.width * c0.height
    mcfg = MOTION_CFG(morph=cfg.get("morph", 0), method=cfg.get("method", 0))
    K, Wm = args.steps, args.warmup
    fill = W_DEFAULT - 1
    e2e_steps = 0 if args.no_e2e else args.e2e_steps
    e2e_warm = 10 if e2e_steps else 0
    # the per-stage pass replays the timed frames on a second handle
    prof_steps = K
    # the clip has 300 frames: shrink the e2e leg to fit
    spare = CLIP_FRAMES - (fill + Wm + K)
    assert spare >= 0, f"--steps + --warmup must leave the {fill} fill frames inside the {CLIP_FRAMES}-frame clip"
    e2e_steps = max(0, min(e2e_steps, spare - e2e_warm))
    if e2e_steps == 0:
        e2e_warm = 0
    n_frames = fill + Wm + K + e2e_warm + e2e_steps
    stream = torch.cuda.Stream(device=dev)
    frames = device_frames(clips, n_frames, stream.cuda_stream)
    st = trb.Streams(S, c0.width, c0.height, 1, mcfg, SEG_CFG(), TRACKER_CFG(), device=local_rank)
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
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    w0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(K):
        st.step_device(ptrs[t], stream.cuda_stream)
        launches += st.last_launches
        t += 1
    st.join(stream.cuda_stream)  # the last step's tracking (internal stream) is inside the timed region
    ev1.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
    clk = clocks.stop(w0, w1)
    frames_job = sum_over_ranks(S * K, world, dev)
    value = aggregate_fps(frames_job, ms / 1e3)

    # ---- per-stage kernel times and the tracker's window pixels (its
    #      algorithmic frame reads) on the SAME frames as the timed steps: a
    #      second handle replays the fill + warm-up frames, then the K timed
    #      frames with CUDA events between the stages
    api.debug_stats(reset=True)
    stage_ms = np.zeros(4)
    track_px = 0.0
    if prof_steps:
        t_timed = fill + Wm
        st2 = trb.Streams(S, c0.width, c0.height, 1, mcfg, SEG_CFG(), TRACKER_CFG(), device=local_rank)
        with torch.cuda.stream(stream):
            for k in range(t_timed):
                st2.step_device(ptrs[k], stream.cuda_stream)
        torch.cuda.synchronize()
        api.debug_stats(reset=True)
        st2.profile(True)
        with torch.cuda.stream(stream):
            for k in range(t_timed, t_timed + prof_steps):
                st2.step_device(ptrs[k], stream.cuda_stream)
        torch.cuda.synchronize()
        stage_ms, n_prof = st2.profile_read()
        st2.profile(False)
        stage_ms = stage_ms / max(1, n_prof)
        track_px = api.debug_stats(reset=True).get("meanshift_window_px", 0) / max(1, n_prof)
        del st2
    t_dev_end = t

    # ---- e2e: the public host API (pinned host frames in, per-step results
    #      out), after a host-path warm-up, >= 100 steps on the wall clock
    e2e = None
    if e2e_steps:
        n_host = e2e_warm + e2e_steps
        pin_t0 = time.perf_counter()
        host = torch.empty((n_host, S, px), dtype=torch.uint8).pin_memory()
        for k in range(n_host):  # each step's S frames back to back, as a capture ring hands them over
            host[k].copy_(frames[:, t + k])
        pin_s = time.perf_counter() - pin_t0
        hn = host.numpy()
        outs = [api.StepOutput(S, blob_cap=64, log_cap=32) for _ in range(n_host)]
        # measured H2D bandwidth of one step's frames (pinned -> HBM)
        probe = torch.empty((S, px), dtype=torch.uint8, device=dev)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for _ in range(3):
            probe.copy_(host[0], non_blocking=True)
        torch.cuda.synchronize()
        h2d_gbs = 3 * S * px / (time.perf_counter() - h0) / 1e9
        del probe
        for k in range(e2e_warm):
            st.step_host_async([hn[k, s] for s in range(S)], outs[k], stream.cuda_stream)
        st.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        for k in range(e2e_warm, n_host):
            st.step_host_async([hn[k, s] for s in range(S)], outs[k], stream.cuda_stream)
        st.synchronize()
        secs = max_over_ranks(time.perf_counter() - e0, world, dev)
        t += n_host
        # the results really came back: every step's blob counts are plausible
        assert all(int(o.n_blobs.max()) > 0 for o in outs[e2e_warm:])
        e2e = {"value": aggregate_fps(sum_over_ranks(S * e2e_steps, world, dev), secs), "unit": "frames/s",
               "h2d_bytes_per_step": S * px, "d2h_bytes_per_step": outs[0].nbytes, "steps": e2e_steps,
               "warmup_steps": e2e_warm, "api": "trb_streams_step_host_async_out (pinned host frames, per-step "
                                                "blob tables + the frame's track-log entries back)",
               "frames": f"clip frames {t - n_host + e2e_warm}..{t - 1} (after the device-timed ones)",
               "h2d_gbs_measured": h2d_gbs, "pin_setup_s": pin_s, "host": bind_info,
               "note": "wall clock over the host-path steps; H2D of a step overlaps the previous step's kernels"}
        del host, hn
    st.synchronize()

    # ---- verify: logs of the first few streams == the reference's (same frames)
    verify = None
    if args.verify_streams and rank == 0 and cfg.get("morph", 0) == 0:
        nv = min(args.verify_streams, S)
        logs = [st.log(s) for s in range(nv)]
        ok, n_entries = verify_logs(clips[:nv], logs, t, mcfg)
        verify = {"streams": nv, "frames": t, "log_entries": n_entries, "identical_to_reference": all(ok)}
        if not all(ok):
            print(f"[bench] VERIFY FAILED: track logs differ from the reference on streams "
                  f"{[i for i, o in enumerate(ok) if not o]}", file=sys.stderr)

    # ---- morphology kernel alone (C2M runs it inside the step; this times
    #      back-to-back launches on the step's masks for its roofline)
    roofline_morph = None
    if first and name == "C5":
        mask0, _ = st.device_planes(0)
        morph_out = torch.empty((S, px), dtype=torch.uint8, device=dev)
        with torch.cuda.stream(stream):
            for _ in range(3):
                api.morph_device(mask0, morph_out.data_ptr(), c0.width, c0.height, S, 3, stream.cuda_stream)
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for _ in range(K):
                api.morph_device(mask0, morph_out.data_ptr(), c0.width, c0.height, S, 3, stream.cuda_stream)
            m1.record(stream)
        torch.cuda.synchronize()
        morph_ms = m0.elapsed_time(m1) / K
        peak, peak_kind = measured_peaks()
        a = MORPH_BYTES_PER_PX * S * px / (morph_ms / 1e3) / 1e9
        roofline_morph = {"bound": "hbm", "kernel": "morph_strip_kernel<open> (erode+dilate fused)", "achieved": a,
                          "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": a / peak,
                          "frac_nominal_8tbs": a / HBM_NOMINAL_GBS,
                          "bytes_per_launch": MORPH_BYTES_PER_PX * S * px, "ms_per_launch": morph_ms,
                          "note": "back-to-back launches on the step's masks; C2M times it inside the step"}
        del morph_out
    del frames
    st = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    peak, peak_kind = measured_peaks()

    def dram_traffic(fname):  # ncu dram bytes per launch, when captured for this workload
        try:
            with open(os.path.join(ROOT, "profiles", fname)) as f:
                d = json.load(f)
            return d["dram_bytes_per_launch"] if d.get("streams") == S and d.get("config", "C5") == name else None
        except Exception:
            return None

    motion_ms = stage_ms[0]
    mode = cfg.get("method", 0) == 1
    mb = ((MODE_BYTES_PER_PX if mode else MOTION_BYTES_PER_PX) + (2 if cfg.get("morph") else 0)) * S * px
    ma = mb / (motion_ms / 1e3) / 1e9 if motion_ms > 0 else 0.0
    # the Mean kernel: motion_mean_bulk_kernel for gray frames with 16-byte
    # aligned planes (bench frames are), W <= 257 (u16 sums), TRB_MOTION_BULK unset/1
    bulk = W_DEFAULT <= 257 and os.environ.get("TRB_MOTION_BULK", "1") != "0"
    mean_kernel = "motion_mean_bulk_kernel" if bulk else "motion_mean_kernel"
    roofline_motion = {"bound": "hbm", "kernel": ("motion_mode_inc_kernel" if mode else mean_kernel) +
                       (" + morph_strip_kernel" if cfg.get("morph") else ""),
                       "achieved": ma, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": ma / peak,
                       "frac_nominal_8tbs": ma / HBM_NOMINAL_GBS,
                       "traffic": dram_traffic("motion_dram_bytes.json"), "bytes_per_launch": mb,
                       "ms_per_step": motion_ms}
    ms_ms = stage_ms[2]
    ms_achieved = track_px / (ms_ms / 1e3) / 1e9 if ms_ms > 0 else 0.0
    stage_names = ["motion", "ccl_stats", "track_meanshift", "track_gate_spawn"]
    dominant = stage_names[int(np.argmax(stage_ms))] if prof_steps else "unknown"
    roofline = {"bound": "hbm", "kernel": "track_meanshift_kernel", "achieved": ms_achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": ms_achieved / peak,
                "frac_nominal_8tbs": ms_achieved / HBM_NOMINAL_GBS,
                "traffic": dram_traffic("meanshift_dram_bytes.json"), "bytes_per_launch": track_px,
                "ms_per_step": ms_ms, "dominant_stage": dominant,
                "algorithmic_bytes": "SURVEY §8(d): window px x iterations x channels (1 B) of frame reads",
                "note": "exact-order fp64 sums (sequential-sum reproduction) make this kernel latency/barrier "
                        "bound, not bandwidth bound; DESIGN.md 3.4"}
    path_gbs = PATH_BYTES_PER_PX * S * world * px / (ms / K / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if args.streams_total else "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": cfg["desc"], "name": name, "width": c0.width, "height": c0.height,
                   "streams_per_gpu": S, "streams_total": int(sum_over_ranks(S, world, dev)), "window": W_DEFAULT,
                   "threshold": 25, "connectivity": 8, "min_area": 4, "k_clusters": 16,
                   "morph": "open" if cfg.get("morph") else "none",
                   "parallelism": f"streams sharded over {world} GPU(s), no collective",
                   "l2": (f"inputs larger than L2 ({S * 4 * px / 1e6:.0f} MB of ring traffic per step)"
                          if S * 4 * px > 126e6 else
                          f"working set per step {S * 12 * px / 1e6:.1f} MB < L2 (126 MB): steps may hit L2"),
                   "stage_ms_per_step": dict(zip(stage_names, [float(x) for x in stage_ms])),
                   "track_window_px_per_step": track_px,
                   "stage_timing": "the timed frames replayed on a second handle with CUDA events between stages",
                   "path_hbm_frac": path_gbs / peak},
        "roofline": roofline, "roofline_motion": roofline_motion,
        "gpu_launches": launches, "clocks": clk,
    }
    if roofline_morph:
        line["roofline_morph"] = roofline_morph
    if e2e:
        line["e2e"] = e2e
    if verify:
        line["verify"] = verify
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if _HOST_AFFINITY:
            os.sched_setaffinity(0, _HOST_AFFINITY)  # the reference baseline gets every host core
        if cfg["recipe"] == "C5":
            threads = args.cpu_threads or os.cpu_count() or 1
            fps, done, secs = run_reference_streams(clips, threads, 2, 0, mcfg)
            line["cpu_baseline"] = {
                "value": fps, "unit": "frames/s", "cores": threads, "kind": "reference",
                "sample": f"{S} C5 streams x 2 steady frames after the {W_DEFAULT - 1}-frame fill on {threads} host "
                          f"threads (nproc {os.cpu_count()}), one stream per thread at a time; {cpu_model()}"}
            one = reference_single_thread(clips[0], CPU_STEADY["C3"], mcfg)
            line["cpu_baseline"]["single_thread_one_stream"] = one
        else:
            line["cpu_baseline"] = reference_single_thread(clips[0], CPU_STEADY[name], mcfg if cfg.get("morph")
                                                           else None)
            if cfg.get("morph"):
                line["cpu_baseline"]["note"] = "the reference has no morphology: its path without it"
    return line


def ours_main(args, rank, world, local_rank):
    bind_info = bind_to_gpu_numa_node(local_rank)
    import torch
    torch.cuda.set_device(local_rank)
    names = ["C1", "C2", "C2M", "C3", "C4", "C5MODE", "C5"] if args.config == "all" else [args.config]
    for i, name in enumerate(names):
        if name not in CONFIGS:
            raise SystemExit(f"unknown --config {name}")
        line = ours_config(args, name, rank, world, local_rank, bind_info, first=(i == len(names) - 1))
        if rank == 0:
            print(json.dumps(line), flush=True)


def dry_main(args, rank, world):
    """Plumbing check without kernels (CPU, gloo): which streams each rank
    owns and the world size the launcher produced."""
    import torch
    import torch.distributed as dist
    cfg = CONFIGS["C5" if args.config == "all" else args.config]
    mine = shard(rank, world, args.streams or cfg["streams"], args.streams_total)
    if world > 1:
        got = [None] * world
        dist.all_gather_object(got, mine)
    else:
        got = [mine]
    t = max_over_ranks(float(rank + 1), world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "shards": got, "max_over_ranks": t}), flush=True)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(argv, args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        print(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    if args.impl == "reference":
        reference_main(args, rank, world)
        return
    import torch
    if world > 1:
        import torch.distributed as dist
        if args.dry_run or not torch.cuda.is_available():
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.dry_run:
            dry_main(args, rank, world)
        else:
            ours_main(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
