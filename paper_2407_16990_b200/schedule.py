"""The launch configuration bench.py times, shared with the full-size parity tests so that both run
exactly the same schedule: two Pipelines (double-buffered state); on one CUDA stream the index path
(regen_select_mbs + regen_pack_regions) of batch k+1 followed by its bilinear pixels
(regen_scatter_bilinear: needs only the frames and the MB owners), while on another the SR of batch
k (regen_enhance_owned) runs; the K steps are captured once into a CUDA graph and replayed. Pure
orchestration over the ABI calls (no arithmetic)."""
from __future__ import annotations

import torch

from . import Pipeline


class PipelinedRunner:
    def __init__(self, make_pipe, device, bilinear: str = "side"):
        """bilinear: where regen_scatter_bilinear of a batch runs — "side" (its own lowest-priority
        stream after the batch's index path), "front" (the index stream) or "back" (the SR stream)."""
        assert bilinear in ("side", "front", "back")
        self.bilinear = bilinear
        self.dev = torch.device(device)
        self.pipes: list[Pipeline] = [make_pipe(), make_pipe()]
        # priorities: the index path (a chain of small latency-bound kernels) highest, so its CTAs are
        # dispatched as soon as the SR kernels' CTAs free an SM; the SR stream next; the bilinear pass
        # (HBM filler that co-runs beside the persistent SR CTAs) lowest
        least, greatest = torch.cuda.Stream.priority_range()
        mid = min(least, greatest + 1)
        self.s_front = torch.cuda.Stream(self.dev, priority=greatest)
        self.s_back = torch.cuda.Stream(self.dev, priority=mid)
        self.s_side = torch.cuda.Stream(self.dev, priority=least)
        self.front_done = [torch.cuda.Event() for _ in range(2)]
        self.back_done = [torch.cuda.Event() for _ in range(2)]
        self.side_done = [torch.cuda.Event() for _ in range(2)]

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
            q = self.pipes[k % 2]
            imp_k, fr_k = ins[k % len(ins)]
            with torch.cuda.stream(self.s_front):
                if not (capturing and k < 2):
                    self.s_front.wait_event(self.back_done[k % 2])   # buffers of batch k-2 are free
                    if self.bilinear == "side":
                        self.s_front.wait_event(self.side_done[k % 2])
                q.select(imp_k, stream=self.s_front)
                q.pack_step(imp_k, stream=self.s_front)
                self.front_done[k % 2].record(self.s_front)
                if self.bilinear == "front":
                    q.scatter_bilinear(fr_k, stream=self.s_front)
            if self.bilinear == "side":
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[k % 2])
                    q.scatter_bilinear(fr_k, stream=self.s_side)
                    self.side_done[k % 2].record(self.s_side)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[k % 2])
                q.enhance_owned(fr_k, stream=self.s_back)
                if self.bilinear == "back":
                    q.scatter_bilinear(fr_k, stream=self.s_back)
                self.back_done[k % 2].record(self.s_back)

    def run_eager(self, imp, frames, n_steps: int, stream=None):
        stream = stream or torch.cuda.current_stream(self.dev)
        for st in (self.s_front, self.s_back, self.s_side):
            st.wait_stream(stream)
        self.steps(imp, frames, n_steps)
        for st in (self.s_front, self.s_back, self.s_side):
            stream.wait_stream(st)

    def capture(self, imp, frames, n_steps: int) -> torch.cuda.CUDAGraph:
        """One CUDA graph holding n_steps pipelined steps (fork/join on a capture stream)."""
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for st in (self.s_front, self.s_back, self.s_side):
                st.wait_stream(cap)
            self.steps(imp, frames, n_steps, capturing=True)
            for st in (self.s_front, self.s_back, self.s_side):
                cap.wait_stream(st)
        return g

    def e2e(self, imp_pin, fr_pin, out_pin, n_steps: int, stream=None) -> float:
        """End-to-end pipelined throughput through the public calls: per step, H2D of the step's inputs
        from pinned host memory (copy stream), the index path (index stream), the bilinear pixels (on
        the stream `self.bilinear` names, as in steps()), the SR pixels (SR stream), and D2H of the step's HR frames into pinned host memory (copy-out stream);
        step k's copies overlap the compute of steps k-1 / k+1. Double-buffered device inputs and host
        outputs (out_pin: two pinned tensors shaped like Pipeline.out). Returns device ms per step."""
        dev = self.dev
        stream = stream or torch.cuda.current_stream(dev)
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        ins = self._inputs(imp_pin, fr_pin)   # pinned host inputs of every selection group of the rank
        imp_d = [torch.empty(ins[0][0].shape, dtype=ins[0][0].dtype, device=dev) for _ in range(2)]
        fr_d = [torch.empty(ins[0][1].shape, dtype=ins[0][1].dtype, device=dev) for _ in range(2)]
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        bil_done = [torch.cuda.Event() for _ in range(2)]
        d2h_done = [torch.cuda.Event() for _ in range(2)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        t0.record(stream)
        for st in (s_h2d, s_d2h, self.s_front, self.s_back, self.s_side):
            st.wait_stream(stream)
        for k in range(n_steps * len(ins)):
            b = k % 2
            q = self.pipes[b]
            imp_pin, fr_pin = ins[k % len(ins)]
            with torch.cuda.stream(s_h2d):
                if k >= 2:
                    # step k-2 no longer reads these inputs: its SR (back) and its bilinear pass
                    s_h2d.wait_event(self.back_done[b])
                    s_h2d.wait_event(bil_done[b])
                imp_d[b].copy_(imp_pin, non_blocking=True)
                fr_d[b].copy_(fr_pin, non_blocking=True)
                h2d_done[b].record(s_h2d)
            with torch.cuda.stream(self.s_front):
                self.s_front.wait_event(h2d_done[b])
                if k >= 2:
                    self.s_front.wait_event(d2h_done[b])   # step k-2's frames have left the device
                q.select(imp_d[b], stream=self.s_front)
                q.pack_step(imp_d[b], stream=self.s_front)
                self.front_done[b].record(self.s_front)
                if self.bilinear == "front":
                    q.scatter_bilinear(fr_d[b], stream=self.s_front)
                    bil_done[b].record(self.s_front)
            if self.bilinear == "side":
                with torch.cuda.stream(self.s_side):
                    self.s_side.wait_event(self.front_done[b])
                    q.scatter_bilinear(fr_d[b], stream=self.s_side)
                    bil_done[b].record(self.s_side)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                q.enhance_owned(fr_d[b], stream=self.s_back)
                if self.bilinear == "back":
                    q.scatter_bilinear(fr_d[b], stream=self.s_back)
                    bil_done[b].record(self.s_back)
                self.back_done[b].record(self.s_back)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(self.back_done[b])
                s_d2h.wait_event(bil_done[b])
                out_pin[b].copy_(q.out, non_blocking=True)
                d2h_done[b].record(s_d2h)
        for st in (s_h2d, s_d2h, self.s_front, self.s_back, self.s_side):
            stream.wait_stream(st)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        return t0.elapsed_time(t1) / n_steps
