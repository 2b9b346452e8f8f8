"""Row-parallel TP MLP forward across GPUs at the Llama-3-8B MLP shape
(BASELINE configs[3]: h4096, ffn14336, bf16, T tokens): the fused push
all-reduce (dist_linear mode "push") against the NCCL baseline (mode "nccl")
and the two GEMMs alone (no all-reduce: the floor).  Device-timed with CUDA
events, max over ranks, modes interleaved over rounds.

    torchrun --nproc-per-node N scripts/tp_forward_bench.py [tokens rounds layout out_dtype]
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist_linear import TpMlpForward  # noqa: E402
from paper_2504_06095_b200.linear import mm  # noqa: E402
from paper_2504_06095_b200.shardmap import build_shard_map  # noqa: E402
from paper_2504_06095_b200.tpnumerics import assignment_from_comp, assignment_from_sync  # noqa: E402


def dmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    layout = sys.argv[3] if len(sys.argv) > 3 else "sync"
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, n = dist.get_rank(), dist.get_world_size()
    h, k = 4096, 14336
    cols = (assignment_from_sync(build_shard_map(k, n + 1, n)) if layout == "sync"
            else assignment_from_comp(build_shard_map(k, n, max(1, n - 1))))
    rng = np.random.default_rng(0)
    A = rng.standard_normal((h, k), dtype=np.float32) / np.sqrt(h)
    B = rng.standard_normal((k, h), dtype=np.float32) / np.sqrt(k)
    odt = {"f32": torch.float32, "bf16": torch.bfloat16}[sys.argv[4] if len(sys.argv) > 4 else "f32"]
    push = TpMlpForward(A, B, cols, T, local, mode="push", out_dtype=odt)
    nccl = TpMlpForward(A, B, cols, T, local, mode="nccl", out_dtype=odt)
    X = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    sh = push.shard
    Zl = torch.empty(T, h, device="cuda", dtype=odt)

    def gemms():
        sh.activations(X)
        mm(sh.Y[:, :sh.n], sh.W[:, 1, :].T, Zl)

    modes = {"push": lambda: push.forward(X), "nccl": lambda: nccl.forward(X), "gemms_only": gemms}
    iters = 20
    res = {m: [] for m in modes}
    for _ in range(rounds):
        for name, fn in modes.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[name].append(dmax(e0.elapsed_time(e1) / iters))
    assert push.status() == 0
    diff = (push.forward(X) - nccl.forward(X)).abs().max().item()
    flops = 2 * 2 * T * h * sh.n
    zbytes = T * h * (4 if odt == torch.float32 else 2)
    if rank == 0:
        out = {"what": f"TP MLP forward across GPUs, Llama-3-8B MLP shape, bf16 GEMMs, {odt} Z",
               "n_gpus": n, "tokens": T, "hidden": h, "ffn": k, "layout": layout,
               "cols_per_rank": [len(c) for c in cols], "rounds": rounds, "iters": iters,
               "median_ms": {m: round(float(np.median(v)), 4) for m, v in res.items()},
               "min_ms": {m: round(float(np.min(v)), 4) for m, v in res.items()},
               "all_ms": {m: [round(x, 4) for x in v] for m, v in res.items()},
               "gemm_tflops_rank0": round(flops / (np.median(res["gemms_only"]) * 1e-3) / 1e12, 1),
               "allreduce_bytes": zbytes,
               "push_vs_nccl_max_abs_diff": diff}
        out["comm_exposed_ms"] = {m: round(out["median_ms"][m] - out["median_ms"]["gemms_only"], 4)
                                  for m in ("push", "nccl")}
        print(json.dumps(out, indent=1), flush=True)
    push.close()
    nccl.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
