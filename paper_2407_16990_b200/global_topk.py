"""Exact cross-rank global top-N (include/regen.h regen_topk_*): the paper's queue
"aggregates and sorts MBs from all streams" taken over the streams of every rank. Four rounds
of a 65536-bin digit histogram (libregen kernels), each summed over the ranks with one all-reduce
(torch.distributed: NCCL over NVLink on GPUs), then the selection of the MBs whose unique global key
is >= the N-th key. Orchestration only: every histogram, digit pick and selection runs in libregen."""
from __future__ import annotations

from . import Pipeline, TOPK_DIGITS, TOPK_STATE_BYTES, topk_histogram, topk_init, topk_pick


class GlobalTopK:
    """State of one rank's part of the protocol: the 24-byte device state and the histogram buffer.

    `allreduce(hist)` sums the int32 histogram over the ranks in place on the current stream; the
    default uses torch.distributed (identity without a process group / with one rank)."""

    def __init__(self, device, allreduce=None, group=None):
        import torch
        self.torch = torch
        self.state = torch.zeros(TOPK_STATE_BYTES, dtype=torch.uint8, device=device)
        self.hist = torch.zeros(TOPK_DIGITS, dtype=torch.int32, device=device)
        self.group = group
        self.allreduce = allreduce or self._dist_allreduce

    def _dist_allreduce(self, hist):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=self.group)

    def find(self, k_total: int, calls, stream=None):
        """calls: [(geom, stream0, importance)] of this rank (its selection groups). Leaves the N-th
        largest global key in self.state (every rank the same)."""
        torch = self.torch
        st = stream or torch.cuda.current_stream(self.hist.device)
        with torch.cuda.stream(st):
            topk_init(k_total, self.state, st)
            for _ in range(4):
                self.hist.zero_()
                for geom, stream0, imp in calls:
                    topk_histogram(geom, stream0, imp, self.state, self.hist, st)
                self.allreduce(self.hist)
                topk_pick(self.hist, self.state, st)

    def select(self, pipe: Pipeline, importance, stream0: int, stream=None):
        """a1 + a2 of one call with the global selection (regen_select_mbs_global)."""
        pipe.select_global(importance, self.state, stream0, stream)


def global_select(pipes_and_inputs, k_total: int, device, allreduce=None, stream=None) -> GlobalTopK:
    """Convenience: [(pipe, stream0, importance)] of this rank -> every pipe selected with the job-wide
    top-k_total (and its regions), ready for pack_step."""
    g = GlobalTopK(device, allreduce)
    g.find(k_total, [(p.geom, s0, imp) for p, s0, imp in pipes_and_inputs], stream)
    for p, s0, imp in pipes_and_inputs:
        g.select(p, imp, s0, stream)
    return g
