"""The degraded-replica backward step with the gradient sync overlapped
(north_star: <= 5 % step overhead over uniform TP).

Per layer, in backward order, the tcgen05 GEMMs write the layer's weight
gradients into its unit-major arena (linear.MlpShard.backward); the layer's
nonuniform sync (dist.NtpSyncGroup.step -- NVLink peer-memory reduce) then runs
on a high-priority side stream under the next layers' GEMMs.  Defaults are
the best measured configuration (scripts/step_bench.py):

  * the TMA-bulk sync kernel on `sync_ctas` SMs and the persistent GEMMs on the
    rest, so neither waits for the other's CTAs to drain;
  * executor policy "healthy": the degraded GPU, which holds the most units,
    only serves its arena and runs no sync kernel beside its GEMMs;
  * the first layer's sync, which no GEMM is left to hide, runs on every SM
    (``uncap_last``).
"""

from __future__ import annotations

import torch

from . import _lib


class OverlappedBackward:
    """layers[l] = (group, [(shard, grads_view), ...]): the layer's NtpSyncGroup
    and this process's shards with their [n, 2, h] views into the group's
    arenas.  ``run(inputs)`` with inputs[l] = [(X, G), ...] per shard."""

    def __init__(self, layers, w_h: float, w_r: float, *, sync_ctas: int = 16,
                 policy: str = "healthy", device: int | None = None, uncap_last: bool = True):
        self.layers = layers
        self.uncap_last = bool(uncap_last)
        self.w_h, self.w_r = float(w_h), float(w_r)
        self.sync_ctas = int(sync_ctas)
        self.device = torch.cuda.current_device() if device is None else device
        self.side = torch.cuda.Stream(self.device, priority=-1)
        for group, _ in layers:
            if group.policy != policy:
                group.set_policy(policy)
        self.sms = torch.cuda.get_device_properties(self.device).multi_processor_count

    def run(self, inputs, stream=None) -> None:
        """One backward step (all layers, last first) with every layer's sync
        overlapped; stream-ordered on `stream` (default: current).  The sync
        kernel choice and the sync / GEMM CTA caps are library-wide options:
        they are set for the duration of the call and restored to the
        caller's values afterwards (not thread-safe against other threads
        changing them meanwhile)."""
        L = _lib.load()
        main = torch.cuda.current_stream(self.device) if stream is None else stream
        saved = (int(L.ntp_get_option(0)), int(L.ntp_get_option(1)), int(L.ntp_gemm_get_max_ctas()))
        L.ntp_set_option(0, 2)                       # TMA-bulk sync kernel
        L.ntp_set_option(1, self.sync_ctas)          # on sync_ctas SMs ...
        L.ntp_gemm_set_max_ctas(self.sms - self.sync_ctas)  # ... GEMMs on the rest
        try:
            for li in reversed(range(len(self.layers))):
                group, shards = self.layers[li]
                with torch.cuda.stream(main):
                    # prescaled aligned groups: the batch weight rides on the
                    # wgrad GEMMs' alpha and the sync is a plain SUM
                    pre = getattr(group, "prescaled", False)
                    for slot, (sh, grads), (X, G) in zip(group.hosted, shards, inputs[li]):
                        alpha = (self.w_h if slot < group.lay.n1 else self.w_r) if pre else 1.0
                        sh.backward(X, G, grads, alpha=alpha)
                self.side.wait_stream(main)
                if li == 0 and self.uncap_last:
                    L.ntp_set_option(1, 0)  # launched after the last GEMM: every SM
                group.step(self.w_h, self.w_r, self.side)
            main.wait_stream(self.side)
        finally:
            L.ntp_set_option(0, saved[0])
            L.ntp_set_option(1, saved[1])
            L.ntp_gemm_set_max_ctas(saved[2])
