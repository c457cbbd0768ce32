"""The launch configuration bench.py times, shared with the full-size parity tests so that both run
exactly the same schedule: P Pipelines (multi-buffered state; P = 2 by default); the index path
(regen_select_mbs + regen_pack_regions) of each batch on one of NF index streams, its bilinear pixels
(regen_scatter_bilinear: needs only the frames and the MB owners) on a low-priority side stream, and
the SR (regen_enhance_owned) of the batches, in order, on one SR stream. With NF > 1 the index paths of
several selection groups run at once, each packer (a sequential one-CTA kernel) on its own SM, so a
rank with many groups (C4, C5) is not bound by one packer's latency. The K steps are captured once into
a CUDA graph and replayed. Pure orchestration over the ABI calls (no arithmetic)."""
from __future__ import annotations

import torch

from . import Pipeline


class PipelinedRunner:
    def __init__(self, make_pipe, device, bilinear: str = "side", nv12: bool = False, n_pipes: int = 2,
                 n_front: int = 1, split_fold: bool = False):
        """bilinear: where regen_scatter_bilinear of a batch runs — "side" (its own lowest-priority
        stream after the batch's index path), "front" (the index stream) or "back" (the SR stream).
        nv12: the frames are NV12 decoder output, converted (regen_nv12_to_rgb8) on the index stream
        into the pipeline's RGB8 buffer at the start of each batch. n_pipes: pipelines (batch k uses
        pipeline k % n_pipes, so up to n_pipes - 1 batches' index paths run ahead of the SR);
        n_front: index streams (batch k's index path on stream k % n_front). split_fold: the SR stream
        runs regen_enhance_partials and the side stream, after the batch's bilinear pass, the fold's
        partial-sum combine (regen_fold_combine_frames), beside the next batch's convolutions."""
        assert bilinear in ("side", "front", "back")
        assert not split_fold or bilinear == "side"
        self.split_fold = split_fold
        assert n_pipes >= 2 and 1 <= n_front <= n_pipes
        self.bilinear = bilinear
        self.nv12 = nv12
        self.dev = torch.device(device)
        self.P = n_pipes
        self.pipes: list[Pipeline] = [make_pipe() for _ in range(n_pipes)]
        # priorities: the index path (a chain of small latency-bound kernels) highest, so its CTAs are
        # dispatched as soon as the SR kernels' CTAs free an SM; the SR stream next; the bilinear pass
        # (HBM filler that co-runs beside the persistent SR CTAs) lowest
        least, greatest = torch.cuda.Stream.priority_range()
        mid = min(least, greatest + 1)
        self.s_fronts = [torch.cuda.Stream(self.dev, priority=greatest) for _ in range(n_front)]
        self.s_front = self.s_fronts[0]
        self.s_back = torch.cuda.Stream(self.dev, priority=mid)
        self.s_side = torch.cuda.Stream(self.dev, priority=least)
        self.front_done = [torch.cuda.Event() for _ in range(n_pipes)]
        self.back_done = [torch.cuda.Event() for _ in range(n_pipes)]
        self.side_done = [torch.cuda.Event() for _ in range(n_pipes)]

    def _streams(self):
        return [*self.s_fronts, self.s_back, self.s_side]

    @staticmethod
    def _inputs(imp, frames):
        """One (importance, frames) pair or lists of them (the selection groups of a rank): batch k of
        a run uses pair k % len."""
        if isinstance(imp, (list, tuple)):
            assert len(imp) == len(frames) and len(imp) > 0
            return list(zip(imp, frames))
        return [(imp, frames)]

    def steps(self, imp, frames, n_steps: int, capturing: bool = False):
        """Enqueue n_steps pipelined steps; a step is one batch of every input pair (each batch: select
        -> pack -> enhance+scatter of one selection group)."""
        ins = self._inputs(imp, frames)
        for k in range(n_steps * len(ins)):
            b = k % self.P
            q = self.pipes[b]
            imp_k, fr_k = ins[k % len(ins)]
            sf = self.s_fronts[k % len(self.s_fronts)]
            with torch.cuda.stream(sf):
                if not (capturing and k < self.P):
                    sf.wait_event(self.back_done[b])   # the pipeline's previous batch is finished
                    if self.bilinear == "side":
                        sf.wait_event(self.side_done[b])
                if self.nv12:
                    fr_k = q.convert_nv12(fr_k, stream=sf)
                q.select(imp_k, stream=sf)
                q.pack_step(imp_k, stream=sf)
                self.front_done[b].record(sf)
                if self.bilinear == "front":
                    q.scatter_bilinear(fr_k, stream=sf)
            if self.bilinear == "side" and not self.split_fold:
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[b])
                    q.scatter_bilinear(fr_k, stream=self.s_side)
                    self.side_done[b].record(self.s_side)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                if self.split_fold:
                    q.enhance_partials(fr_k, stream=self.s_back)
                else:
                    q.enhance_owned(fr_k, stream=self.s_back)
                if self.bilinear == "back":
                    q.scatter_bilinear(fr_k, stream=self.s_back)
                self.back_done[b].record(self.s_back)
            if self.split_fold:
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[b])
                    q.scatter_bilinear(fr_k, stream=self.s_side)
                    self.s_side.wait_event(self.back_done[b])
                    q.fold_combine(stream=self.s_side)
                    self.side_done[b].record(self.s_side)

    def run_eager(self, imp, frames, n_steps: int, stream=None):
        stream = stream or torch.cuda.current_stream(self.dev)
        for st in self._streams():
            st.wait_stream(stream)
        self.steps(imp, frames, n_steps)
        for st in self._streams():
            stream.wait_stream(st)

    def capture(self, imp, frames, n_steps: int) -> torch.cuda.CUDAGraph:
        """One CUDA graph holding n_steps pipelined steps (fork/join on a capture stream)."""
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for st in self._streams():
                st.wait_stream(cap)
            self.steps(imp, frames, n_steps, capturing=True)
            for st in self._streams():
                cap.wait_stream(st)
        return g

    def e2e(self, imp_pin, fr_pin, out_pin, n_steps: int, stream=None) -> float:
        """End-to-end pipelined throughput through the public calls: per batch, H2D of the batch's inputs
        from pinned host memory (copy stream), the index path (an index stream), the bilinear pixels (on
        the stream `self.bilinear` names, as in steps()), the SR pixels (SR stream), and D2H of the
        batch's HR frames into pinned host memory (copy-out stream); a batch's copies overlap the
        compute of the others. Device inputs per pipeline, two pinned host outputs (out_pin: shaped like
        Pipeline.out). Returns device ms per step (a step = one batch of every input pair)."""
        dev = self.dev
        stream = stream or torch.cuda.current_stream(dev)
        P = self.P
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        ins = self._inputs(imp_pin, fr_pin)   # pinned host inputs of every selection group of the rank
        imp_d = [torch.empty(ins[0][0].shape, dtype=ins[0][0].dtype, device=dev) for _ in range(P)]
        fr_d = [torch.empty(ins[0][1].shape, dtype=ins[0][1].dtype, device=dev) for _ in range(P)]
        h2d_done = [torch.cuda.Event() for _ in range(P)]
        bil_done = [torch.cuda.Event() for _ in range(P)]
        d2h_done = [torch.cuda.Event() for _ in range(P)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        t0.record(stream)
        streams = [s_h2d, s_d2h, *self._streams()]
        for st in streams:
            st.wait_stream(stream)
        for k in range(n_steps * len(ins)):
            b = k % P
            q = self.pipes[b]
            imp_pin, fr_pin = ins[k % len(ins)]
            sf = self.s_fronts[k % len(self.s_fronts)]
            with torch.cuda.stream(s_h2d):
                if k >= P:
                    # the batch that last used these device inputs is done with them: its SR (back)
                    # and its bilinear pass
                    s_h2d.wait_event(self.back_done[b])
                    s_h2d.wait_event(bil_done[b])
                imp_d[b].copy_(imp_pin, non_blocking=True)
                fr_d[b].copy_(fr_pin, non_blocking=True)
                h2d_done[b].record(s_h2d)
            with torch.cuda.stream(sf):
                sf.wait_event(h2d_done[b])
                if k >= P:
                    sf.wait_event(d2h_done[b])   # the pipeline's previous frames have left the device
                fr_b = q.convert_nv12(fr_d[b], stream=sf) if self.nv12 else fr_d[b]
                q.select(imp_d[b], stream=sf)
                q.pack_step(imp_d[b], stream=sf)
                self.front_done[b].record(sf)
                if self.bilinear == "front":
                    q.scatter_bilinear(fr_b, stream=sf)
                    bil_done[b].record(sf)
            if self.bilinear == "side" and not self.split_fold:
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[b])
                    q.scatter_bilinear(fr_b, stream=self.s_side)
                    bil_done[b].record(self.s_side)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                if self.split_fold:
                    q.enhance_partials(fr_b, stream=self.s_back)
                else:
                    q.enhance_owned(fr_b, stream=self.s_back)
                if self.bilinear == "back":
                    q.scatter_bilinear(fr_b, stream=self.s_back)
                    bil_done[b].record(self.s_back)
                self.back_done[b].record(self.s_back)
            if self.split_fold:   # the bilinear pass and the fold's combine; bil_done = the batch's frames complete
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[b])
                    q.scatter_bilinear(fr_b, stream=self.s_side)
                    self.s_side.wait_event(self.back_done[b])
                    q.fold_combine(stream=self.s_side)
                    bil_done[b].record(self.s_side)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(self.back_done[b])
                s_d2h.wait_event(bil_done[b])
                out_pin[k % 2].copy_(q.out, non_blocking=True)
                d2h_done[b].record(s_d2h)
        for st in streams:
            stream.wait_stream(st)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        return t0.elapsed_time(t1) / n_steps
