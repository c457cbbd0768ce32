#!/usr/bin/env python
"""Benchmark of the RegenHance region-aware enhancement hot path on B200.

One step = one pass of the whole hot path (select -> pack -> enhance -> scatter, SURVEY §8(a) rows
a1-a8) over one batch of synthetic input per selection group the rank owns. Default workload: the
BASELINE.json configs[1] C2 (1 stream x 30 frames 640x360 -> 1920x1080, top-20% MBs, EDSR 8
resblocks / 32 ch bf16), one group per rank (weak scaling). `--config c4`: the 64-stream job of
configs[3] (8 selection groups of 8 streams, top-15%) sharded over the ranks (strong scaling);
`--config c5 --ratio R`: configs[4] (16 streams of 720p, 8 groups of 2, EDSR 16 x 64, ratio R%).
Inputs are resident in HBM when the timed region starts; the K timed steps run back to back (the
index path of batch k+1 overlapped with the SR of batch k on a second CUDA stream, double-buffered
state) as one captured CUDA graph; each step's working set is >10x the L2.
Multi-GPU: one process per GPU. `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (NCCL); each rank enhances its own selection groups (no data-path
collective); NCCL only reduces the elapsed time (MAX) and frame counts (SUM) after the timed loop.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5] [--ratio R]
                  [--impl ours|reference]
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

import synth  # noqa: E402

METRIC = "enhanced frames/sec at 360p→1080p (device-timed, max over ranks)"


def executed_flops_per_lr_px(sr: synth.SRConfig) -> int:
    """FLOPs the BF16 tensor-core network executes per LR box pixel: the UP∘TAIL fold
    replaces the last upsampler conv + HR tail by one LR conv C -> 3(p+2)^2 (p = last shuffle factor)."""
    C, s = sr.channels, sr.scale
    if sr.n_resblocks == 0 or not sr.bf16:
        return sr_flops_per_lr_px(sr)
    f = 2 * 9 * 3 * C + (2 * sr.n_resblocks + 1) * 2 * 9 * C * C
    p = s
    if s == 4:
        f += 2 * 9 * C * 4 * C
        p = 2
    return f + 2 * 9 * C * 3 * (p + 2) ** 2 * (4 if s == 4 else 1)


# kernels that run as one CTA (the sequential packer, the per-segment selection, the one-CTA sort and
# list builder): a long one occupies one SM beside the full-GPU kernels, so it is not the GPU's dominant
# kernel even when its launch time is the largest (C4: the packers of 3 groups in flight)
ONE_CTA_KERNELS = {"pack", "pack_policy", "select", "sort_rank", "stitch_lists"}


def dominant_kernel(kern: dict) -> str:
    """Name with the largest summed device time among the kernels that spread over the GPU."""
    wide = {k: v for k, v in kern.items() if k not in ONE_CTA_KERNELS} or kern
    return max(wide.items(), key=lambda kv: kv[1][1])[0]


def sr_flops_per_lr_px(sr: synth.SRConfig) -> int:
    """Useful FLOPs (2 per MAC) of the SR network per LR box pixel."""
    C, s = sr.channels, sr.scale
    if sr.n_resblocks == 0:
        return 2 * 9 * 3 * C + 2 * 9 * C * 3 * s * s
    f = 2 * 9 * 3 * C + (2 * sr.n_resblocks + 1) * 2 * 9 * C * C
    if s == 4:
        f += 2 * 9 * C * 4 * C + 4 * 2 * 9 * C * 4 * C
    else:
        f += 2 * 9 * C * C * s * s
    f += s * s * 2 * 9 * C * 3
    return f


def load_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)["kernels"].get(kernel)
    except Exception:
        return None


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled every ~0.5 ms from
    a thread (nvidia-smi's 100 ms loop would see a 30 ms region once or never); nvidia-smi fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.sm: list[float] = []
        self.mask = 0
        self.max_mhz = None
        self.stop = threading.Event()
        self.t = None
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))

    def _loop(self):
        while not self.stop.is_set():
            try:
                self.sample()
            except Exception:
                return
            time.sleep(0.0005)

    def __exit__(self, *a):
        self.stop.set()
        if self.t is not None:
            self.t.join(timeout=2)
        if self.nv is not None:
            try:
                self.sample()
            except Exception:
                pass
        else:   # fallback: one nvidia-smi reading right after the region
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits",
                                      "-i", str(self.gpu)], capture_output=True, text=True, timeout=20).stdout
                sm, mx = (float(v) for v in out.strip().split(","))
                self.sm.append(sm)
                self.max_mhz = mx
            except Exception:
                pass

    def summary(self) -> dict:
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm),
                "source": "nvml" if self.nv is not None else "nvidia-smi after the region"}


# --------------------------------------------------------------------------------- CPU oracle

def cpu_oracle_frames(wl: synth.Workload, seed: int, n_frames: int, threads: int, s0: int = 0,
                      u8: bool = False) -> dict:
    """The oracle as it stands (C, fp64) doing the complete hot path for the first `n_frames` frames
    of one selection-group batch: the index path of the whole batch (selection is over the group,
    P:641), stitch, the SR of every placed box of those frames, and their HR frames (scatter). The
    per-box SR and per-frame scatter run on `threads` host threads (ref_enhance_mt / ref_scatter_mt:
    the same single-threaded functions distributed over POSIX threads). Returns frames/s measured on
    whole frames (no extrapolation)."""
    import oracle
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, seed, s0=s0)
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, seed, s0=s0)
    w64 = oracle.sr_weights_for(wl.sr, synth.sr_weights(wl.sr, 0))
    t0 = time.perf_counter()
    ip = oracle.index_path(imp, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                           max_bins=wl.max_bins)
    lr = oracle.gather(fr, ip["boxes"], ip["placement"], wl.bin_w, wl.bin_h, ip["num_bins"], wl.sr.bf16)
    flat = ip["boxes"][:, 0].astype(np.int64) * wl.F + ip["boxes"][:, 1]
    mine = np.flatnonzero((flat < n_frames) & (ip["placement"][:, 0] >= 0))
    pl = ip["placement"].copy()
    keep = np.zeros(len(pl), bool)
    keep[mine] = True
    pl[~keep, 0] = -1          # boxes of other frames: not enhanced in this sample
    hr = oracle.enhance(wl.sr, w64, lr, ip["boxes"], pl, threads=threads)
    out = oracle.scatter(fr, ip["boxes"], ip["placement"], ip["owner"], hr, wl.sr.scale, wl.bin_w, wl.bin_h, 0,
                         n_frames, threads=threads)
    if u8:
        oracle.quantize_u8(fr, ip["owner"], out, wl.sr.scale, 0, n_frames)
    dt = time.perf_counter() - t0
    return {"value": n_frames / dt, "unit": "frames/s", "cores": threads, "kind": "oracle",
            "sample": f"complete hot path of frames 0..{n_frames - 1} of one {wl.S}x{wl.F}-frame {wl.name} batch "
                      f"(index path of the whole batch, SR of their {len(mine)} boxes, their "
                      f"{'u8 ' if u8 else ''}HR frames) in "
                      f"{dt:.1f} s on {threads} host threads",
            "seconds": dt}


def _oracle_frames_for(wl: synth.Workload, seconds: float, threads: int) -> int:
    """Frames of a bounded sample taking ~`seconds` on `threads` cores (the oracle's SR costs about
    1.2e9 FLOP/s per core, measured on the dev box)."""
    per_frame = sr_flops_per_lr_px(wl.sr) * wl.W * wl.H * wl.pct / 100 * 1.45 / 1.2e9 / threads + 0.01
    return int(max(1, min(wl.S * wl.F, round(seconds / per_frame))))


def run_reference(args, wl: synth.Workload) -> None:
    """The reference arm: the paper has no runnable code, so the reference is the CPU oracle as it
    stands, on all host cores, on the same workload/metric (rank 0 only under torchrun)."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = oracle.host_cores()
    nfr = _oracle_frames_for(wl, 4.0, threads)
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_frames(wl, seed=i % 3, n_frames=1 if i < args.warmup else nfr, threads=threads,
                              u8=args.out == "u8")
        if i >= args.warmup:
            vals.append(r["value"])
            last = r
    v = statistics.mean(vals)
    cb = dict(last)
    cb.pop("seconds", None)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * nfr / v,
            "higher_is_better": True, "scaling": "weak" if wl.groups == 0 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name + ("_u8out" if args.out == "u8" else ""), "frames_per_step": nfr,
                       "sample": cb["sample"]},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------- launcher

def _relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) started as a plain process: re-run this script as N ranks (one per GPU)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def rank_env(args) -> tuple[int, int, int]:
    """(world, rank, local rank) of this process; validates --gpus against a torchrun environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def job_groups(wl: synth.Workload, world: int, rank: int) -> list[tuple[int, int]]:
    """Stream ranges of the selection groups this rank enhances (shard.py): weak configs give every
    rank one group (streams rank*S ..), fixed-size jobs (C4, C5) shard their groups contiguously."""
    from paper_2407_16990_b200 import shard
    n_groups = wl.groups if wl.groups > 0 else world
    return shard.rank_groups(n_groups * wl.S, wl.S, world, rank)


# --------------------------------------------------------------------------------- our arm

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--ratio", type=float, default=None, help="importance ratio in %% (C5 sweep: 5..50)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--dry-run", action="store_true", help="launcher/sharding only (CPU, gloo): print the plan")
    ap.add_argument("--out", default="bf16", choices=["bf16", "u8"],
                    help="HR frame type: the model dtype (bf16), or u8 codes (reading D20: clamp, round half to even)")
    ap.add_argument("--input", default="rgb", choices=["rgb", "nv12"],
                    help="frame format: RGB8, or NV12 decoder output converted on the GPU inside the step")
    args = ap.parse_args()
    wl = synth.CONFIGS[args.config]
    if args.ratio is not None:
        import dataclasses
        wl = dataclasses.replace(wl, pct=args.ratio, name=f"{wl.name}_r{args.ratio:g}")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args, wl)
        return
    world, rank, local = rank_env(args)
    groups = job_groups(wl, world, rank)
    if args.dry_run:
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
        from paper_2407_16990_b200 import shard
        t, f = shard.reduce_timing(1.0 + rank, float(len(groups) * wl.S * wl.F))
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "config": wl.name, "rank0_groups": groups,
                              "max_ms": t, "frames": f}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    import paper_2407_16990_b200 as rg
    from paper_2407_16990_b200 import shard
    from paper_2407_16990_b200.schedule import PipelinedRunner

    seed = 0
    G = len(groups)
    imp_h = [synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, seed, s0=g0) for g0, _ in groups]
    nv12 = args.input == "nv12"
    fr_h = [(synth.frames_nv12 if nv12 else synth.frames_rgb8)(wl.S, wl.F, wl.H, wl.W, seed, s0=g0) for g0, _ in groups]
    w = synth.sr_weights(wl.sr, 0)

    def make_pipe():
        return rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h,
                           max_bins=wl.max_bins, partition_mb=wl.partition_mb, scale=wl.sr.scale,
                           channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks, weights=w, bf16=wl.sr.bf16,
                           res_scale=wl.sr.res_scale, device=dev, frame_format=rg.FORMAT_NV12 if nv12 else rg.FORMAT_RGB8,
                           out_dtype=rg.DTYPE_U8 if args.out == "u8" else None)

    frames_step = G * wl.S * wl.F          # this rank's frames per step
    stream = torch.cuda.current_stream(dev)
    kern_all, kern, n_warm, graph = {}, {}, 1, None
    total_ms, stage, box_px, exec_px, sel_px, n_bins, n_boxes = 0.0, np.zeros(3), 0, 0, 0, 0, 0
    e2e_t = float("nan")
    clk_summary = None
    if G > 0:
        # two pipelines (double-buffered state): the index path (select + pack) of batch k+1 on one CUDA
        # stream while the SR (enhance + scatter) of batch k runs on another (schedule.py: the same
        # runner the full-size parity tests drive); a rank with several groups cycles through them
        # up to 4 pipelines, the index paths of up to 3 batches (consecutive groups, or consecutive chunks of
        # one group) in flight at once, each packer on its own SM, so that a sequential packer that is
        # slower than a batch's SR (8-stream groups) does not bound the step; memory permitting
        # (REGEN_PIPES / REGEN_FRONTS override, A/B aids)
        free0 = torch.cuda.mem_get_info(dev)[0]
        probe = make_pipe()
        per_pipe = max(1, free0 - torch.cuda.mem_get_info(dev)[0])
        del probe
        torch.cuda.empty_cache()
        n_pipes = int(max(2, min(4, (0.7 * torch.cuda.mem_get_info(dev)[0]) // per_pipe)))
        n_pipes = int(os.environ.get("REGEN_PIPES", n_pipes))
        n_front = int(os.environ.get("REGEN_FRONTS", max(1, n_pipes - 1)))
        split = os.environ.get("REGEN_SPLIT_FOLD", "0") == "1"
        runner = PipelinedRunner(make_pipe, dev, bilinear=os.environ.get("REGEN_BILINEAR", "side"),
                                 n_pipes=n_pipes, n_front=n_front, split_fold=split)
        pipes = runner.pipes
        p = pipes[0]
        imp = [torch.from_numpy(a).to(dev) for a in imp_h]
        fr = [torch.from_numpy(a).to(dev) for a in fr_h]
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

        def step_instrumented(gi):
            ev[0].record(stream)
            frames = fr[gi]   # RGB8, or NV12 read directly by the gather and the bilinear pass
            p.select(imp[gi])
            ev[1].record(stream)
            p.pack_step(imp[gi])
            ev[2].record(stream)
            p.enhance_scatter(frames)
            ev[3].record(stream)

        # serial instrumented batches (L2 flushed before each): per-stage device time and the work of
        # every group (box pixels, bins) for the roofline
        n_instr = max(1, min(args.steps, 3))
        for gi in range(G):
            for it in range(max(args.warmup, 1) + n_instr):
                flush.zero_()
                step_instrumented(gi)
                torch.cuda.synchronize()
                if it >= max(args.warmup, 1):
                    stage += [ev[i].elapsed_time(ev[i + 1]) / n_instr for i in range(3)]
            res = p.host_results()
            assert res["status"] == 0, f"device status {res['status']}"
            bx = res["boxes"]
            placed = bx["bin"] >= 0
            box_px += int((bx["w"][placed].astype(np.int64) * bx["h"][placed]).sum())
            sel_px += int((res["owner"] >= 0).sum()) * 256
            n_bins += res["num_bins"]
            n_boxes += int(placed.sum())
        runner.run_eager(imp, fr, max(args.warmup, 2))     # warm the pipelined schedule
        torch.cuda.synchronize()

        # The K timed steps are one CUDA graph (captured once, replayed): no host launch overhead between
        # the ~50 kernels of a batch. A warm replay with every libregen launch bracketed by CUDA events on
        # its own stream (regen_trace_*) gives the per-kernel table and names the dominant kernel; in the
        # timed replay only the dominant kernel's launches are bracketed (its live device time for the
        # roofline) so the event nodes barely perturb the step.
        def capture(n_steps: int, trace_prefix):
            if trace_prefix is not None:
                rg.trace_filter(trace_prefix or None)
                rg.trace_enable(True)
            g = runner.capture(imp, fr, n_steps)
            rg.trace_enable(False)
            rg.trace_filter(None)
            return g

        rg.trace_read()
        if not args.no_graph:
            n_warm = max(args.warmup, 3)
            warm = capture(n_warm, "")     # all kernels traced
            warm.replay()
            torch.cuda.synchronize()
            for name, ms in rg.trace_read():
                k = kern_all.setdefault(name, [0, 0.0])
                k[0] += 1
                k[1] += ms
            dom_name = dominant_kernel(kern_all)
            graph = capture(args.steps, dom_name)   # its trace records are read after the timed replay
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if G > 0:
        if graph is None:
            rg.trace_enable(True)
        with ClockSampler(local) as clk:
            t0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                runner.run_eager(imp, fr, args.steps, stream)
            t1.record(stream)
            torch.cuda.synchronize()
        clk_summary = clk.summary()
        rg.trace_enable(False)
        total_ms = t0.elapsed_time(t1)
        for name, ms in rg.trace_read():
            k = kern.setdefault(name, [0, 0.0])
            k[0] += 1
            k[1] += ms
        for q in pipes:
            assert q.host_results()["status"] == 0
    if world > 1:
        dist.barrier()
    total_ms, frames = shard.reduce_timing(total_ms, frames_step * args.steps, device=dev)
    value = frames / (total_ms / 1000.0)

    # e2e through the public API with host buffers: every batch H2D-copies its inputs from pinned host
    # memory, runs the four calls and D2H-copies its HR frames into pinned host memory; batches are
    # pipelined (copies of batch k overlap compute of batches k-1 / k+1, schedule.PipelinedRunner.e2e),
    # the device time from the first H2D to the last D2H divided by the steps
    h2d_step = sum(a.nbytes for a in imp_h) + sum(a.nbytes for a in fr_h)
    d2h_step = 0
    if G > 0 and args.e2e_steps > 0:
        imp_pin = [torch.from_numpy(a).pin_memory() for a in imp_h]
        fr_pin = [torch.from_numpy(a).pin_memory() for a in fr_h]
        out_pin = [torch.empty(p.out.shape, dtype=p.out.dtype).pin_memory() for _ in range(2)]
        d2h_step = G * int(p.out.numel() * p.out.element_size())
        runner.e2e(imp_pin, fr_pin, out_pin, 1, stream)                   # warm
        e2e_t = runner.e2e(imp_pin, fr_pin, out_pin, args.e2e_steps, stream)
        last = args.e2e_steps * G - 1
        assert torch.equal(out_pin[last % 2], pipes[last % runner.P].out.cpu())
    if world > 1:
        t = torch.tensor([0.0 if e2e_t != e2e_t else e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
        # whole-job work for the roofline: every rank's box pixels / bins
        wk = torch.tensor([box_px, sel_px, n_bins, n_boxes, frames_step], dtype=torch.float64, device=dev)
        dist.all_reduce(wk, op=dist.ReduceOp.SUM)
        job_box_px, job_sel_px, job_bins, job_boxes, job_frames = (float(v) for v in wk.tolist())
    else:
        job_box_px, job_sel_px, job_bins, job_boxes, job_frames = box_px, sel_px, n_bins, n_boxes, frames_step
    e2e_val = job_frames / (e2e_t / 1000.0)

    if not kern_all:   # no graph: the timed region itself traced every kernel
        kern_all, n_warm = kern, args.steps
    if rank == 0:
        peaks = load_peaks()
        fp = sr_flops_per_lr_px(wl.sr)
        fe = executed_flops_per_lr_px(wl.sr)
        flops_step = job_box_px * fp            # SURVEY §8(d) FLOP_box of the whole job per step
        peak_b, peak_s = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        # dominant kernel = largest share of the summed device time (warm traced replay); its live
        # launch times come from the timed region (rank 0's)
        roof = {}
        if kern:
            dom = dominant_kernel(kern)
            dom_n, dom_ms_total = kern[dom]
            dom_ms = dom_ms_total / dom_n
            C = wl.sr.channels
            per_px = {"resblock": 2 * 2 * 9 * C * C, "conv_res_a": 2 * 9 * C * C, "conv_res_b": 2 * 9 * C * C,
                      "conv_body": 2 * 9 * C * C}
            if dom in per_px:
                alg = per_px[dom] * box_px / G    # algorithmic FLOPs per launch: per-LR-box-pixel x box px per batch
                achieved = alg / (dom_ms / 1000.0) / 1e12
                peak = peak_b if wl.sr.bf16 else fp32_peak
                roof = {"kernel": dom, "bound": "tensor" if wl.sr.bf16 else "alu", "achieved": achieved, "peak": peak,
                        "unit": "TFLOP/s", "frac": achieved / peak, "traffic": load_traffic(dom),
                        "peak_sustained": peak_s if wl.sr.bf16 else None,
                        "frac_vs_sustained": achieved / peak_s if wl.sr.bf16 else None,
                        "algorithmic_per_launch": alg,
                        "per_unit": f"{per_px[dom]} FLOP per LR box pixel x {box_px / G:.0f} box px per batch",
                        "launch_ms_mean": dom_ms,
                        "peak_source": (f"{peaks['source']} bf16 burst (the kernel runs in a {total_ms:.0f} ms region; "
                                        "the sustained 4-s matmul peak is the second field)") if wl.sr.bf16
                        else "fp32 FMA 148x128x2x1.965GHz"}
            else:
                roof = {"kernel": dom, "bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                        "traffic": load_traffic(dom), "launch_ms_mean": dom_ms}
            occ_bin = job_box_px / max(job_bins * wl.bin_w * wl.bin_h, 1)
            if roof.get("frac") is not None and occ_bin > 0:
                # the kernel computes every pixel of the bins it covers: the same time over the FLOPs of
                # the bin pixels (frac / box-over-bin fill) is the tensor-core work rate it executes
                roof["frac_bin_px"] = roof["frac"] / occ_bin
            roof.update({"flops_per_step": flops_step, "box_px_per_step": job_box_px,
                         "occupy_ratio_sel_over_box": job_sel_px / max(job_box_px, 1),
                         "occupy_ratio_box_over_bin": occ_bin,
                         "sr_network_tflops": box_px * fp / (stage[2] / 1000.0) / 1e12 if stage[2] else None})
        # HBM-bound kernels against the measured copy bandwidth: algorithmic bytes per launch / mean
        # launch time (concurrent replay: includes co-scheduling with the SR stream)
        es_out = 1 if args.out == "u8" else (2 if wl.sr.bf16 else 4)
        s2 = wl.sr.scale * wl.sr.scale
        lr_bytes = wl.S * wl.F * wl.W * wl.H * 3
        hbm_alg = {"scatter_bilinear": ((s2 * (wl.S * wl.F * wl.W * wl.H * G - sel_px) * 3 * es_out) / max(G, 1)
                                        + lr_bytes, "HR bytes of the non-owned pixels written + LR frames read"),
                   "stitch": ((box_px * 3 + n_bins * wl.bin_w * wl.bin_h * 16) / max(G, 1),
                              "box pixels read (u8 RGB) + packed bins written (8 bf16 channels); the bin map, "
                              "owned-pixel destinations and occupancy bits it also writes are implementation traffic")}
        hbm = {}
        for name, (nbytes, what) in hbm_alg.items():
            if name in kern_all:
                ms = kern_all[name][1] / kern_all[name][0]
                gbs = nbytes / (ms / 1000.0) / 1e9
                hbm[name] = {"algorithmic_bytes": int(nbytes), "what": what, "ms_mean_concurrent": ms,
                             "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
                             "traffic": load_traffic(name)}
        # whole-step roofline: the slower of the packed-conv FLOPs (box pixels x FLOP per LR
        # pixel) at the tensor peak and the algorithmic bytes (LR frames + importance read, HR frames
        # written) at the copy bandwidth; also with the FLOPs the folded network executes
        bytes_alg = job_frames * (wl.W * wl.H * 3 + 4 * wl.GH * wl.GW + s2 * wl.W * wl.H * 3 * es_out)
        ms_step = total_ms / args.steps
        t_hbm = bytes_alg / (peaks["hbm_gbs"] * 1e9) * 1e3 / world
        def step_frac(flops, pk):
            t_tc = flops / (pk * 1e12) * 1e3 / world      # the job's work spread over the ranks
            return max(t_tc, t_hbm), t_tc
        pk = peak_b if wl.sr.bf16 else fp32_peak
        t_roof, t_tc = step_frac(flops_step, pk)
        t_roof_s, _ = step_frac(flops_step, peak_s if wl.sr.bf16 else fp32_peak)
        t_roof_e, t_tc_e = step_frac(job_box_px * fe, pk)
        step_roof = {"bound": "tensor" if t_tc >= t_hbm else "hbm", "flops_per_step": flops_step,
                     "flop_per_lr_box_px": fp, "executed_flop_per_lr_box_px": fe,
                     "executed_flops_per_step": job_box_px * fe,
                     "bytes_alg_per_step": bytes_alg, "t_tensor_ms": t_tc, "t_hbm_ms": t_hbm,
                     "roof_value": job_frames / (t_roof / 1e3), "frac": t_roof / ms_step,
                     "frac_vs_sustained": t_roof_s / ms_step,
                     "frac_executed": t_roof_e / ms_step,
                     "note": "frac: survey FLOP_box at the burst tensor peak; frac_vs_sustained: same at the 4-s "
                             "sustained peak; frac_executed: the FLOPs the folded network actually executes"}
        kernels = {name: {"launches_per_step": n / n_warm, "ms_mean": ms / n,
                          "share": ms / sum(v[1] for v in kern_all.values())} for name, (n, ms) in
                   sorted(kern_all.items(), key=lambda kv: -kv[1][1])}
        strong = wl.groups > 0
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "bf16" if wl.sr.bf16 else "f32", "data": "synthetic",
            "config": {"workload": wl.name + ("_nv12" if nv12 else "") + ("_u8out" if args.out == "u8" else ""),
                       "input": "NV12 (BT.601 fused into the gather and the bilinear pass)" if nv12 else "RGB8",
                       "output": "u8 HR frames (D20: clamp, round half to even)" if args.out == "u8"
                       else ("bf16" if wl.sr.bf16 else "fp32") + " HR frames", "streams_total": (wl.groups if strong else world) * wl.S,
                       "selection_group_streams": wl.S, "groups_rank0": G, "frames_per_step": int(job_frames),
                       "frame": f"{wl.W}x{wl.H}->x{wl.sr.scale}", "topk_pct": wl.pct,
                       "bins_per_step": int(job_bins), "bin": f"{wl.bin_w}x{wl.bin_h}", "boxes_per_step": int(job_boxes),
                       "sr": f"EDSR {wl.sr.n_resblocks}x{wl.sr.channels} x{wl.sr.scale}",
                       "l2": "timed steps run back to back; each step's working set (packed activations and HR "
                             "frames, >1 GB) is >10x the 126 MB L2, so no step finds the previous one's data",
                       "schedule": (f"{runner.P if G else 0} pipelines, index paths (select+pack) of up to "
                                    f"{len(runner.s_fronts) if G else 0} batches on their own streams ahead of the SR "
                                    "(enhance+scatter) stream, bilinear pass on a lowest-priority stream; a rank cycles "
                                    "through its selection groups")
                                   + ("; the K steps replayed as one captured CUDA graph" if graph is not None else ""),
                       "parallelism": (f"strong dp{world}: {wl.groups} selection groups sharded by rank" if strong
                                       else f"weak dp{world}: one selection group per rank") +
                                      ", no data-path collective"},
            "stages_ms": {"select": stage[0] / max(G, 1), "pack": stage[1] / max(G, 1),
                          "enhance_scatter": stage[2] / max(G, 1),
                          "note": "per batch (one selection group), serial instrumented, L2 flushed before each"},
            "roofline": roof,
            "roofline_hbm_kernels": hbm,
            "roofline_step": step_roof,
            "kernels": kernels,
            "kernels_note": "device ms per launch from a warm replay of the same captured schedule with every libregen "
                            "launch bracketed by CUDA events on its stream (concurrent streams: times include "
                            "co-scheduling); the roofline kernel's time is from the timed replay",
            "e2e": {"value": e2e_val, "unit": "frames/s", "ms_per_step": e2e_t, "steps": args.e2e_steps,
                    "schedule": "public calls per batch with pinned-host H2D of inputs and D2H of the HR frames "
                                "inside the timed region; batches pipelined on 4 streams (copies overlap compute)",
                    "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step},
            "gpu_launches": int(round(sum(v[0] for v in kern_all.values()) / n_warm * args.steps)),
            "clocks": clk_summary,
        }
        if not args.no_cpu_baseline:
            import oracle
            th = oracle.host_cores()
            cb = cpu_oracle_frames(wl, seed, _oracle_frames_for(wl, 12.0, th), th, s0=groups[0][0] if groups else 0,
                                   u8=args.out == "u8")
            cb.pop("seconds", None)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
