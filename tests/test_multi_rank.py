"""Multi-rank host logic on CPU (gloo, world_size 2): selection-group sharding (shard.py, SURVEY
§8(e)) gives every group to exactly one rank, the per-group results do not depend on the world size
(checked with the oracle's index path, bit for bit), and the measurement's reductions are MAX of
the elapsed time and SUM of the frames."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2407_16990_b200 import shard

N_STREAMS, GROUP, F, W, H = 6, 2, 2, 160, 96
K_PCT = 20.0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _group_result(s0: int, s1: int) -> dict:
    GW, GH = synth.grid(W, H)
    imp = synth.importance_maps(s1 - s0, F, GH, GW, 3, "blobs", s0=s0)
    k = int((s1 - s0) * F * GH * GW * K_PCT // 100)
    ip = oracle.index_path(imp, W, H, k, partition_mb=3, bin_w=64, bin_h=64, max_bins=64)
    return {"sel": ip["sel"].tobytes(), "boxes": ip["boxes"].tobytes(), "placement": ip["placement"].tobytes(),
            "owner": ip["owner"].tobytes(), "num_bins": int(ip["num_bins"])}


def _worker(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = {g: _group_result(*g) for g in shard.rank_groups(N_STREAMS, GROUP, world, rank)}
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        t, f = shard.reduce_timing(10.0 * (rank + 1), 30.0 * (rank + 1), device="cpu")
        if rank == 0:
            merged = {}
            for part in gathered:
                for g, v in part.items():
                    assert g not in merged, f"group {g} computed twice"
                    merged[g] = v
            q.put((merged, t, f))
    finally:
        dist.destroy_process_group()


def test_group_and_rank_slices():
    assert shard.group_bounds(5, 2) == [(0, 2), (2, 4), (4, 5)]
    assert shard.group_bounds(0, 8) == []
    # balanced contiguous shares cover every item exactly once
    for n in range(0, 20):
        for world in range(1, 9):
            spans = [shard.rank_slice(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    # C4: 64 streams = 8 groups of 8 -> 8/4/2/1 groups per rank at 1/2/4/8 ranks
    for world in (1, 2, 4, 8):
        assert all(len(shard.rank_groups(64, 8, world, r)) == 8 // world for r in range(world))
    with pytest.raises(ValueError):
        shard.rank_slice(4, 2, 2)


def test_sharded_results_identical_for_any_world_size():
    """world_size 2 over gloo vs world_size 1 in-process: same groups, bit-identical index path."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, t, f = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 20.0 and f == 90.0          # MAX of 10, 20; SUM of 30, 60
    single = {g: _group_result(*g) for g in shard.rank_groups(N_STREAMS, GROUP, 1, 0)}
    assert sorted(merged) == sorted(single) == shard.group_bounds(N_STREAMS, GROUP)
    for g in single:
        for key in single[g]:
            assert merged[g][key] == single[g][key], f"group {g}: {key} differs"


def test_group_maps_are_slices_of_the_global_workload():
    """A shard's inputs equal the same streams of the whole workload (seeded by global stream index)."""
    GW, GH = synth.grid(W, H)
    full = synth.importance_maps(N_STREAMS, F, GH, GW, 3, "blobs")
    frames = synth.frames_rgb8(N_STREAMS, F, 8, 8, 3)
    for s0, s1 in shard.group_bounds(N_STREAMS, GROUP):
        np.testing.assert_array_equal(synth.importance_maps(s1 - s0, F, GH, GW, 3, "blobs", s0=s0), full[s0:s1])
        np.testing.assert_array_equal(synth.frames_rgb8(s1 - s0, F, 8, 8, 3, s0=s0), frames[s0:s1])


def _bench_dry_run(*args):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", *args], capture_output=True,
                         text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_bench_launcher_spawns_its_own_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself as 2 ranks (gloo in the
    dry run): C4's 8 selection groups split 4/4 (strong scaling), C2 gives each rank one group (weak),
    and the MAX/SUM reductions see both ranks."""
    d = _bench_dry_run("--gpus", "2", "--config", "c4")
    assert d["n_gpus"] == 2 and d["rank0_groups"] == [[0, 8], [8, 16], [16, 24], [24, 32]]
    assert d["max_ms"] == 2.0 and d["frames"] == 64 * 30
    d = _bench_dry_run("--gpus", "2")
    assert d["n_gpus"] == 2 and d["rank0_groups"] == [[0, 1]] and d["frames"] == 2 * 30
    d = _bench_dry_run("--config", "c5")
    assert d["n_gpus"] == 1 and len(d["rank0_groups"]) == 8 and d["frames"] == 16 * 30


# ------------------------------------------------------------------ exact cross-rank global top-N

def _keys(imp: np.ndarray, stream0: int) -> np.ndarray:
    """Reading D2/D17 keys with global ids: ord(score) << 32 | (0xFFFFFFFF - gid), written out in numpy
    (the protocol's CPU stand-in for the libregen histogram kernel)."""
    b = imp.astype(np.float32).reshape(-1).copy()
    b[b == 0] = 0.0                                     # -0 == +0
    u = b.view(np.uint32).astype(np.uint64)
    ordv = np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)
    ordv = np.where(np.isnan(b), 0, ordv).astype(np.uint64)
    gid = np.arange(b.size, dtype=np.uint64) + np.uint64(stream0 * imp[0].size)
    return (ordv << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - gid)


def _topk_worker(rank, world, port, q, k_total):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    try:
        GW, GH = synth.grid(W, H)
        s0, s1 = shard.rank_slice(N_STREAMS, world, rank)
        imp = synth.importance_maps(s1 - s0, F, GH, GW, 7, "levels", s0=s0)
        keys = _keys(imp, s0)
        prefix, k_rem, flag = 0, k_total, "search" if k_total > 0 else "none"
        for rnd in range(4):
            sh, hs = 48 - 16 * rnd, 64 - 16 * rnd
            m = keys if hs == 64 else keys[(keys >> np.uint64(hs)) == np.uint64(prefix >> hs)]
            hist = torch.from_numpy(np.bincount(((m >> np.uint64(sh)) & np.uint64(0xFFFF)).astype(np.int64),
                                                minlength=1 << 16).astype(np.int32))
            dist.all_reduce(hist, op=dist.ReduceOp.SUM)        # the one exchange of the round
            h = hist.numpy().astype(np.int64)
            if flag == "search" and rnd == 0 and k_rem >= h.sum():
                flag = "all"
            if flag == "search":
                above = np.concatenate([np.cumsum(h[::-1])[::-1][1:], [0]])   # keys with a larger digit
                d = int(np.flatnonzero((above < k_rem) & (k_rem <= above + h))[0])
                prefix |= d << sh
                k_rem -= int(above[d])
        sel = (np.ones(keys.size, bool) if flag == "all" else np.zeros(keys.size, bool) if flag == "none"
               else keys >= np.uint64(prefix))
        out = [None] * world
        dist.all_gather_object(out, (s0, sel.reshape(imp.shape).astype(np.uint8)))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k_frac", [(2, 0.2), (3, 0.05), (2, 0.0), (2, 1.5)])
def test_global_topk_protocol_is_exact_over_ranks(world, k_frac):
    """The 4-round 16-bit-digit histogram protocol of SURVEY §8(f)2 (gloo all-reduce between the rounds)
    selects exactly the oracle's GLOBAL top-k over the union of all ranks' streams, with
    massive ties (10 importance levels), for any world size."""
    GW, GH = synth.grid(W, H)
    k_total = int(k_frac * N_STREAMS * F * GH * GW)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_topk_worker, args=(r, world, port, q, k_total)) for r in range(world)]
    for p in ps:
        p.start()
    parts = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    sel = np.concatenate([s for _, s in sorted(parts, key=lambda t: t[0])], 0)
    imp = synth.importance_maps(N_STREAMS, F, GH, GW, 7, "levels")
    ref = oracle.select(imp, W, H, oracle.MODE_TOPK, k_total)
    np.testing.assert_array_equal(sel, ref)
    assert sel.sum() == min(k_total, imp.size)


def test_bench_dominant_kernel_skips_one_cta_kernels():
    """bench.py's roofline kernel: the largest summed device time among the kernels that spread over the
    GPU; a one-CTA kernel (the packer of a C4 group, 12 ms on one SM) does not displace the residual
    block, and is chosen only when nothing else ran."""
    import bench
    kern = {"pack": [8, 93.5], "resblock": [64, 40.7], "scatter_bilinear": [8, 16.4], "select": [8, 4.1]}
    assert bench.dominant_kernel(kern) == "resblock"
    assert bench.dominant_kernel({"pack": [1, 2.0], "select": [1, 1.0]}) == "pack"
    assert bench.dominant_kernel({"conv_fold_frames": [1, 0.2], "resblock": [8, 0.72]}) == "resblock"
