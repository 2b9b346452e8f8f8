"""Host-buffer gradient sync: the call a user of the reference's numpy API makes.

The reference's ``nonuniform_grad_sync`` takes gradients in host memory
(numpy, tpnumerics.py:289) and mutates them in place.  ``HostSync`` is that
boundary for a whole workload: pinned host arenas in, pinned host arenas out,
with the device kernel in between.  Transfers are split into pieces and
pipelined over two copy streams (H2D and D2H run concurrently over PCIe's two
directions) with the sync kernel of piece i overlapping the copies of its
neighbours, so the call is bound by host-link bandwidth, not by the sum of its
stages.
"""

from __future__ import annotations

import torch

from .plans import OPS, Plan, tensor_ptrs


class HostSync:
    def __init__(self, plan: Plan, arena_elems, dtype, device: int = 0, piece_plans=None,
                 back_to_back: bool = False):
        """plan: a finalized plan over the arenas (buffer i = arena i).
        piece_plans: optional [(plan_i, arena_ranges_i)] splitting the work into
        pipelined pieces; arena_ranges_i = [(arena, lo, hi)] element ranges the
        piece reads and writes.

        back_to_back=False (default): every run() is fully ordered on the
        current stream -- its host-to-device copies start after everything the
        caller queued on that stream before the call, and the stream waits for
        its device-to-host copies at the end.  back_to_back=True is for a loop
        of runs over the same host buffers that nothing else touches in
        between: piece i's host-to-device copy then waits only for the previous
        run's device-to-host copy of piece i (not for the whole previous run),
        so both host-link directions stay busy across runs; the current stream
        still waits for each run's device-to-host copies before later work."""
        self.dev = torch.device("cuda", device)
        self.plan = plan if plan.device is not None else plan.upload(device)
        self.arenas = [torch.empty(e, dtype=dtype, device=self.dev) for e in arena_elems]
        self.ptrs = tensor_ptrs(self.arenas)
        self.pieces = piece_plans
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self.launches_per_run = 1 if not piece_plans else len(piece_plans)
        self.back_to_back = bool(back_to_back)
        self._d2h_done = None  # per piece: the previous run's D2H of that piece

    def run(self, host, w_a: float, w_b: float) -> None:
        """host: pinned CPU tensors, one per arena; synced in place (stream-ordered
        on the current stream; synchronize before reading them)."""
        cur = torch.cuda.current_stream(self.dev)
        if not self.pieces:
            for d, h in zip(self.arenas, host):
                d.copy_(h, non_blocking=True)
            self.plan.grad_sync(self.ptrs, OPS["weighted"], w_a, w_b, cur)
            for d, h in zip(self.arenas, host):
                h.copy_(d, non_blocking=True)
            return
        # back_to_back: piece i's H2D waits only for the previous run's D2H of
        # piece i (same host and device ranges), not for the whole previous
        # run, so consecutive runs keep both PCIe directions busy.
        chained = self.back_to_back and self._d2h_done is not None
        if not chained:
            self.h2d.wait_stream(cur)
        done = []
        for i, (plan_i, ranges) in enumerate(self.pieces):
            if chained:
                self.h2d.wait_event(self._d2h_done[i])
            with torch.cuda.stream(self.h2d):
                for a, lo, hi in ranges:
                    self.arenas[a][lo:hi].copy_(host[a][lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.h2d)
            cur.wait_event(ev)
            plan_i.grad_sync(self.ptrs, OPS["weighted"], w_a, w_b, cur)
            ev2 = torch.cuda.Event()
            ev2.record(cur)
            self.d2h.wait_event(ev2)
            with torch.cuda.stream(self.d2h):
                for a, lo, hi in ranges:
                    host[a][lo:hi].copy_(self.arenas[a][lo:hi], non_blocking=True)
            ev3 = torch.cuda.Event()
            ev3.record(self.d2h)
            done.append(ev3)
        self._d2h_done = done
        cur.wait_stream(self.d2h)
