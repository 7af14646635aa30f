"""World-size-2 coverage of the multi-GPU path on CPU (gloo).

bench.py shards independent camera streams over ranks (weak scaling, no
data-path collective) and times the job as the MAX over ranks.  These tests
run that plumbing in two gloo processes: the shards are disjoint and cover
the job, per-rank results equal a single-process run of the same streams
(checked with the CPU oracle on small clips), and the timing reduction /
aggregate are the ones bench.py reports.
"""
import hashlib
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

STREAMS_PER_RANK = 2
N_FRAMES = 14


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _clip(stream: int):
    from paper_1310_3322_b200.synth import mix_seed, random_clip
    return random_clip(64, 48, 3, 6, 10, True, mix_seed(7, stream), mix_seed(1007, stream), N_FRAMES)


def _stream_digest(stream: int) -> str:
    """Oracle pipeline (motion W=9 -> CCL -> tracker) of one small stream."""
    from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
    from tests import _oracle as O
    clip = _clip(stream)
    frames, _ = O.orc_frames(clip)
    mcfg = MOTION_CFG()
    mcfg.window = 9
    out, log, _ = O.run_pipeline_cpu(clip, frames, mcfg, SEG_CFG(), TRACKER_CFG())
    h = hashlib.sha256()
    for t, m, lab, blobs in out:
        h.update(np.int64(t).tobytes())
        h.update(np.ascontiguousarray(m).tobytes())
        h.update(np.ascontiguousarray(lab).tobytes())
        h.update(np.ascontiguousarray(blobs).tobytes())
    h.update(np.ascontiguousarray(log).tobytes())
    assert len(out) == N_FRAMES - 8 and len(log) > 0  # masks every frame after the fill, tracks spawned
    return h.hexdigest()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        mine = bench.shard(rank, world, STREAMS_PER_RANK)
        digests = {s: _stream_digest(s) for s in mine}
        gathered = [None] * world
        dist.all_gather_object(gathered, {"streams": mine, "digests": digests})
        # per-rank "device time": rank r is slower by r ms; the job time is the max
        t = bench.max_over_ranks(10.0 + rank, world)
        frames = bench.sum_over_ranks(STREAMS_PER_RANK * 5, world)
        fps = bench.aggregate_fps(frames, t / 1e3)
        q.put((rank, gathered, t, fps))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    from tests import _oracle as O
    O.build_oracle()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    gathered = res[0][1]
    assert res[1][1] == gathered  # every rank sees the same gather
    owned = [s for g in gathered for s in g["streams"]]
    assert sorted(owned) == list(range(world * STREAMS_PER_RANK))  # disjoint, complete
    # per-rank results are exactly the single-process results of those streams
    for g in gathered:
        for s, d in g["digests"].items():
            assert d == _stream_digest(s)
    # MAX over ranks on every rank, and the aggregate bench.py reports
    for rank, _, t, fps in res:
        assert t == 11.0
        assert fps == pytest.approx(STREAMS_PER_RANK * world * 5 / 0.011)


def test_reference_arm_runs_on_rank0_only(capsys):
    import bench

    args = bench.parse(["--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-threads", "1"])
    bench.reference_main(args, rank=1, world=2)
    assert capsys.readouterr().out == ""


def test_single_rank_helpers():
    import bench
    assert bench.shard(0, 1, 64) == list(range(64))
    assert bench.shard(3, 4, 4) == [12, 13, 14, 15]
    # strong scaling: 64 streams over G GPUs, stream s on GPU floor(s*G/64)
    for g in (1, 2, 4, 8):
        parts = [bench.shard(r, g, 0, 64) for r in range(g)]
        assert sorted(x for p in parts for x in p) == list(range(64))
        assert all(len(p) == 64 // g for p in parts)
        assert all(s * g // 64 == r for r, p in enumerate(parts) for s in p)
    assert bench.max_over_ranks(2.5, 1) == 2.5
    assert bench.aggregate_fps(64 * 20, 0.2) == pytest.approx(6400.0)


@pytest.mark.parametrize("extra,per_rank", [([], 64), (["--streams-total", "64"], 32)])
def test_bench_gpus_flag_launches_that_many_ranks(extra, per_rank):
    """`python bench.py --gpus 2` (no torchrun) re-launches itself with two
    ranks; the ranks report world size 2 and disjoint shards covering the
    job (weak: 64 streams per rank; strong: 64 streams over the job)."""
    import json
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"] + extra,
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    shards = line["shards"]
    assert [len(x) for x in shards] == [per_rank, per_rank]
    assert sorted(shards[0] + shards[1]) == list(range(2 * per_rank if not extra else 64))
    assert line["max_over_ranks"] == 2.0
