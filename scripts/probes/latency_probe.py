"""Per-launch cost of the handshake building blocks (torchrun, N=2), each as
K launches in one CUDA graph: empty kernel, acq_rel / sc system fences, a
relaxed system store to the peer's signal page, fence + store, and raw
ping-pongs (store / poll) with and without the fence.  Kernels in
latency_kernels.cu (built here with nvcc if missing)."""

import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402

SO = os.path.join(HERE, "latency_kernels.so")


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    if rank == 0 and not os.path.exists(SO):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "latency_kernels.cu")],
                       check=True)
    dist.barrier()
    L = ctypes.CDLL(SO)
    L.probe_launch.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    lay = pair_layout(ModelShape("tiny", 64, 8, 0, 1), 4, 3)
    grp = NtpSyncGroup(lay, Placement.default(2, 4, 3), torch.float32, device=local).upload()
    peer_word, own_word = grp.post_ready[0], grp.wait_ready[0]
    K = 200
    s = torch.cuda.Stream()
    out = {}

    def timed_graph(build):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            build()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / K * 1e3], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return round(float(t.item()), 3)

    sp = lambda: ctypes.c_void_p(s.cuda_stream)  # noqa: E731
    for name, which in (("empty", 0), ("fence_acq_rel_sys", 1), ("fence_sc_sys", 2),
                        ("store_relaxed_sys_peer", 3), ("fence_store_peer", 4)):
        out[f"{name}_us"] = timed_graph(lambda w=which: [L.probe_launch(w, peer_word, 1, sp())
                                                          for _ in range(K)])
    base = [1000]
    for name, store in (("pingpong_relaxed", 3), ("pingpong_fenced", 4)):
        b = base[0]

        def build(b=b, store=store):
            for i in range(1, K + 1):
                if rank == 0:
                    L.probe_launch(store, peer_word, b + i, sp())
                    L.probe_launch(5, own_word, b + i, sp())
                else:
                    L.probe_launch(5, own_word, b + i, sp())
                    L.probe_launch(store, peer_word, b + i, sp())
        out[f"{name}_us_per_round_trip"] = timed_graph(build)
        base[0] += 10 * K
    if rank == 0:
        print(json.dumps(out), flush=True)
    grp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
