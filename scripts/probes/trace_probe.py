"""Phase timestamps of the signalled sync kernel (torchrun, N=2): globaltimer
stamps written by CTA 0 / the last CTA (ntp_debug_sync_trace): ready post,
ready seen, last CTA in, done posted, done seen; for a 2-unit plan and a 16 MB
per replica plan, one-launch and three-launch steps."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    L = _lib.load()
    L.ntp_debug_sync_trace.argtypes = [ctypes.c_void_p]
    tr = torch.zeros(8, dtype=torch.int64, device="cuda")
    L.ntp_debug_sync_trace(ctypes.c_void_p(tr.data_ptr()))
    out = {}
    for name, shape in (("tiny", ModelShape("tiny", 64, 8, 0, 1)),
                        ("16MB", ModelShape("s16", 4096, 1024, 0, 1))):
        lay = pair_layout(shape, 4, 3)
        grp = NtpSyncGroup(lay, Placement.default(2, 4, 3), torch.bfloat16, device=local).upload()
        for fused in (True, False):
            grp.fused_step = fused
            rows = []
            for it in range(30):
                tr.zero_()
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                grp.step(4 / 7, 3 / 7)
                e1.record()
                torch.cuda.synchronize()
                t = tr.cpu().numpy().astype(np.int64)
                if it >= 5 and t[0] and t[5]:
                    rows.append([(t[i] - t[0]) / 1e3 for i in range(1, 6)] + [e0.elapsed_time(e1) * 1e3])
            med = np.median(np.array(rows), axis=0).round(2).tolist() if rows else None
            allm = [None] * dist.get_world_size()
            dist.all_gather_object(allm, med)
            out[f"{name}_{'1launch' if fused else '3launch'}"] = {
                "us_since_cta0_start [ready_posted, ready_seen, last_cta_in, done_posted, done_seen, event_total]": allm}
        dist.barrier()
        grp.close()
    L.ntp_debug_sync_trace(None)
    if rank == 0:
        print(json.dumps(out, indent=1), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
