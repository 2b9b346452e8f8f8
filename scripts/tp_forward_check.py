"""Multi-GPU parity of the row-parallel TP MLP forward (torchrun, n ranks).

Every rank holds its uneven column shard of (A, B) from the reference's shard
map, runs dist_linear.TpMlpForward (mode push: the second GEMM's epilogue
pushes partial-sum boxes to the row-block owners over NVLink; or nccl), and
checks Z against the fp64 oracle of mlp_forward_dense (tpnumerics.py:170-185)
on the same bf16-rounded inputs (<= 2e-2), bit-identical across ranks.

    torchrun --nproc-per-node N scripts/tp_forward_check.py [mode layout tokens out_dtype]
layout: "comp" (healthy TP-N columns of build_shard_map(k, N, N-1)) or
"sync" (the degraded replica's contiguous columns of build_shard_map(k, N+1, N))
"""

import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import _procgroup  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2504_06095_b200.dist_linear import TpMlpForward  # noqa: E402
from paper_2504_06095_b200.shardmap import build_shard_map  # noqa: E402
from paper_2504_06095_b200.tpnumerics import assignment_from_comp, assignment_from_sync  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "push"
    layout = sys.argv[2] if len(sys.argv) > 2 else "sync"
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 512
    out_dtype = {"f32": torch.float32, "bf16": torch.bfloat16}[sys.argv[4] if len(sys.argv) > 4 else "f32"]
    os.environ["NCCL_DEBUG"] = "WARN"
    local = _procgroup.init()
    rank, n = dist.get_rank(), dist.get_world_size()
    h, k = 256, 1000
    if layout == "comp":
        cols = assignment_from_comp(build_shard_map(k, n, max(1, n - 1)))
    else:
        cols = assignment_from_sync(build_shard_map(k, n + 1, n))
    rng = np.random.default_rng(9)  # identical on every rank
    r64 = lambda x: torch.from_numpy(x).to(torch.bfloat16).double().numpy()  # noqa: E731
    A, B = r64(rng.standard_normal((h, k)) / np.sqrt(h)), r64(rng.standard_normal((k, h)) / np.sqrt(k))
    tp = TpMlpForward(A, B, cols, T, local, mode=mode, out_dtype=out_dtype)
    ok = True
    for it in range(3):
        X = r64(rng.standard_normal((T, h)))
        Z = tp.forward(torch.from_numpy(X).to(torch.bfloat16).cuda()).clone()
        torch.cuda.synchronize()
        assert tp.status() == 0, "signal timeout"
        want = O.mlp_forward_dense(X, A, B)
        err = O.rel_err(Z.double().cpu().numpy(), want)  # <= 2e-2 (bf16 operands)
        digest = hashlib.sha256(Z.cpu().view(torch.uint8).numpy().tobytes()).hexdigest()
        allz = [None] * n
        dist.all_gather_object(allz, digest)   # bit-identical Z on every rank
        same = all(z == allz[0] for z in allz)
        ok &= err <= 2e-2 and same
        if rank == 0:
            print(f"tp_forward n={n} {mode} {layout} T={T} {out_dtype} iter={it} rel_err={err:.3e} "
                  f"identical={same}", flush=True)
    tp.close()
    if rank == 0:
        print("PASS" if ok else "FAIL", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
