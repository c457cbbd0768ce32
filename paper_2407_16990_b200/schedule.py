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
    def __init__(self, make_pipe, device, bilinear_on_front: bool = True):
        self.bilinear_on_front = bilinear_on_front
        self.dev = torch.device(device)
        self.pipes: list[Pipeline] = [make_pipe(), make_pipe()]
        # the index path is a chain of small latency-bound kernels: give its stream the higher priority
        # so its CTAs are dispatched as soon as the SR kernels' CTAs free an SM
        self.s_front = torch.cuda.Stream(self.dev, priority=-1)
        self.s_back = torch.cuda.Stream(self.dev, priority=0)
        self.front_done = [torch.cuda.Event() for _ in range(2)]
        self.back_done = [torch.cuda.Event() for _ in range(2)]

    def steps(self, imp, frames, n_steps: int, capturing: bool = False):
        """Enqueue n_steps pipelined steps (each: one batch through select -> pack -> enhance+scatter)."""
        for k in range(n_steps):
            q = self.pipes[k % 2]
            with torch.cuda.stream(self.s_front):
                if not (capturing and k < 2):
                    self.s_front.wait_event(self.back_done[k % 2])   # buffers of batch k-2 are free
                q.select(imp, stream=self.s_front)
                q.pack_step(imp, stream=self.s_front)
                self.front_done[k % 2].record(self.s_front)
                if self.bilinear_on_front:
                    q.scatter_bilinear(frames, stream=self.s_front)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[k % 2])
                q.enhance_owned(frames, stream=self.s_back)
                if not self.bilinear_on_front:
                    q.scatter_bilinear(frames, stream=self.s_back)
                self.back_done[k % 2].record(self.s_back)

    def run_eager(self, imp, frames, n_steps: int, stream=None):
        stream = stream or torch.cuda.current_stream(self.dev)
        self.s_front.wait_stream(stream)
        self.s_back.wait_stream(stream)
        self.steps(imp, frames, n_steps)
        stream.wait_stream(self.s_front)
        stream.wait_stream(self.s_back)

    def capture(self, imp, frames, n_steps: int) -> torch.cuda.CUDAGraph:
        """One CUDA graph holding n_steps pipelined steps (fork/join on a capture stream)."""
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            self.s_front.wait_stream(cap)
            self.s_back.wait_stream(cap)
            self.steps(imp, frames, n_steps, capturing=True)
            cap.wait_stream(self.s_front)
            cap.wait_stream(self.s_back)
        return g
