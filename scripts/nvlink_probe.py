"""NVLink peer-memory probe for the push sync (run under torchrun, 2 ranks).

Rank 1 maps rank 0's buffer through CUDA IPC and times, per kernel variant:
  read  : local <- peer      (ntp_reshard, a = peer, b = local)
  write : peer  <- local     (ntp_reshard, a = local, b = peer)
  pair  : both <- w_a*peer + w_b*local   (ntp_grad_sync: read + write over the link)
and a symmetric split where both ranks push half of the pair work at once,
plus symmetric pure reads / writes (both ranks move the whole buffer at once).
GB/s are per link direction.
"""

import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.dist import DeviceOps  # noqa: E402
from paper_2504_06095_b200.plans import OPS, Plan  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    nbytes = int(float(sys.argv[1]) * 2**30) if len(sys.argv) > 1 else 2**30
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    L = _lib.load()
    ops = DeviceOps(local)
    buf = ops.alloc(nbytes)
    tab = [None, None]
    dist.all_gather_object(tab, ops.handle(buf))
    peer = ops.open(tab[1 - rank])
    elems = nbytes // 2  # bf16
    unit = 8192          # 16 KiB units
    n = elems // unit

    def plan(a_buf, b_buf, lo=0, hi=None):
        hi = n if hi is None else hi
        import numpy as np
        idx = np.arange(lo, hi, dtype=np.int64)
        p = Plan(_lib.NTP_BF16)
        p.add_units(unit, np.full(len(idx), a_buf), idx * unit, np.full(len(idx), b_buf), idx * unit)
        return p.finalize().upload(local)

    bufs = [buf, peer]   # index 0 local, 1 peer
    scratch = ops.alloc(nbytes)
    bufs3 = [buf, peer, scratch]
    res = {}
    for vname, v in (("ldg", 1), ("bulk4x1", 2), ("bulk3x2", 3)):
        _lib.check(L.ntp_set_option(0, v))
        r = {}
        if rank == 1:
            p_read, p_write, p_pair = plan(1, 0), plan(0, 1), plan(1, 0)
            ms = timed(lambda: p_read.reshard(bufs))
            r["read_gbs"] = round(nbytes / ms / 1e6, 1)
            ms = timed(lambda: p_write.reshard(bufs))
            r["write_gbs"] = round(nbytes / ms / 1e6, 1)
            ms = timed(lambda: p_pair.grad_sync(bufs, OPS["weighted"], 0.5, 0.5))
            r["pair_gbs_per_direction"] = round(nbytes / ms / 1e6, 1)
        dist.barrier()
        # symmetric: each rank pushes half of the units (rank 0 the first half)
        half = plan(1, 0, 0, n // 2) if rank == 0 else plan(1, 0, n // 2, n)
        torch.cuda.synchronize()
        dist.barrier()
        ms = timed(lambda: half.grad_sync(bufs, OPS["weighted"], 0.5, 0.5))
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        r["symmetric_pair_gbs_per_direction"] = round(nbytes / t.item() / 1e6, 1)
        # symmetric read / write: both ranks move the whole buffer at once
        for name, pl in (("symmetric_read_gbs_per_direction", plan(1, 2)),
                         ("symmetric_write_gbs_per_direction", plan(2, 1))):
            dist.barrier()
            ms = timed(lambda: pl.reshard(bufs3))
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            r[name] = round(nbytes / t.item() / 1e6, 1)
        res[vname] = r
        dist.barrier()
    # reference: torch/NCCL send-recv of the same bytes (one direction)
    x = torch.empty(elems, dtype=torch.bfloat16, device="cuda")

    def sendrecv():
        if rank == 0:
            dist.send(x, 1)
        else:
            dist.recv(x, 0)
    ms = timed(sendrecv, 10)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res["nccl_send_recv_gbs"] = round(nbytes / t.item() / 1e6, 1)
    y = torch.empty(elems, dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: dist.all_reduce(y), 10)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res["nccl_allreduce_busbw_gbs"] = round(nbytes / t.item() / 1e6, 1)
    _lib.check(L.ntp_set_option(0, 0))
    if rank == 1:
        print(json.dumps({"bytes": nbytes, "results": res}, indent=1), flush=True)
    dist.barrier()
    ops.close(peer)
    ops.free(buf)
    ops.free(scratch)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
