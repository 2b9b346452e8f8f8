"""Multi-GPU failure reconfiguration (dist_reconfig.DistReconfig), run under
torchrun.  One GPU of replica D dies; H goes TP-n1 -> comp layout, D's
survivors go TP-n1 -> TP-(n1-1), the dead rank's units pulled from H.

    torchrun --nproc-per-node N scripts/reconfig_check.py check [n1 dead]
        bit-exact check of every destination arena (rank 0 gathers them)
    torchrun --nproc-per-node N scripts/reconfig_check.py bench [n1 dead layers]
        Llama-3-8B-shaped layers, bf16 params + fp32 master / exp_avg / exp_avg_sq;
        device time of the pulls (max over ranks), bytes local / over NVLink
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import _procgroup  # noqa: E402

from paper_2504_06095_b200.dist_reconfig import (DistReconfig, FailureLayout,  # noqa: E402
                                                 failure_placement)
from paper_2504_06095_b200.shardmap import build_shard_map  # noqa: E402
from paper_2504_06095_b200.tpnumerics import (assignment_from_comp,  # noqa: E402
                                              assignment_from_sync, contiguous_assignment)
from paper_2504_06095_b200.workloads import LLAMA3_8B, ModelShape  # noqa: E402

STATES = {"param": torch.bfloat16, "master": torch.float32, "exp_avg": torch.float32,
          "exp_avg_sq": torch.float32}


def segs_of(shape: ModelShape, layers: int):
    return tuple((k, u) for _ in range(layers) for _kind, k, u in shape.segments())


def expected(lay, src):
    """Destination arenas gathered column by column from the source arenas."""
    n1, n2 = lay.n1, lay.n2
    out = {s: np.empty(e, dtype=src[0].dtype) for s, e in enumerate(lay.slot_elems())
           if s >= 2 * n1}
    base = np.zeros(lay.n_slots(), dtype=np.int64)
    for k, unit in lay.segs:
        smap = build_shard_map(k, n1, n2)
        contig = contiguous_assignment(k, n1)
        comp, sync = assignment_from_comp(smap), assignment_from_sync(smap)
        pos = {}
        for name, cols, slot0 in (("c", contig, 0), ("h", comp, 2 * n1), ("d", sync, 3 * n1)):
            for r, cs in enumerate(cols):
                for i, c in enumerate(cs):
                    pos[(name, int(c))] = (slot0 + r, int(base[slot0 + r]) + i * unit)
        for c in range(k):
            hs, ho = pos[("c", c)]
            owner = hs
            ds, do = (hs, ho) if owner == lay.dead else (n1 + hs, int(base[n1 + hs]) + (ho - int(base[hs])))
            ts, to = pos[("h", c)]
            out[ts][to:to + unit] = src[hs][ho:ho + unit]
            ts, to = pos[("d", c)]
            out[ts][to:to + unit] = src[ds][do:do + unit]
        for i in range(n1):
            base[i] += len(contig[i]) * unit
            if i != lay.dead:
                base[n1 + i] += len(contig[i]) * unit
            base[2 * n1 + i] += len(comp[i]) * unit
        for j in range(n2):
            base[3 * n1 + j] += len(sync[j]) * unit
    return out


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "check"
    n1 = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    dead = int(sys.argv[3]) if len(sys.argv) > 3 else n1 - 1
    local = _procgroup.init()
    rank, world = dist.get_rank(), dist.get_world_size()
    if mode == "check":
        shape, layers = ModelShape("check", hidden=64, ffn=1000, heads=8, layers=2), 2
    else:
        shape, layers = LLAMA3_8B, int(sys.argv[4]) if len(sys.argv) > 4 else 2
    lay = FailureLayout(n1, n1 - 1, dead, segs_of(shape, layers))
    proc = failure_placement(n1, dead, world)
    g = DistReconfig(lay, proc, STATES, device=local).upload()
    src_slots = [s for s in g.hosted if s < 2 * n1]
    for name, dt in STATES.items():
        for s in src_slots:
            gen = torch.Generator(device="cuda").manual_seed(1000 * s + len(name))
            a = g.arena(s, name)
            a.copy_(torch.randn(a.numel(), generator=gen, device="cuda").to(dt))
    if mode == "check":
        g.run()
        ok = True
        for name, dt in STATES.items():
            mine = {s: g.arena(s, name).view(torch.int16 if dt == torch.bfloat16 else torch.int32)
                    .cpu().numpy() for s in g.hosted}
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            if rank == 0:
                got = {}
                for d in allv:
                    got.update(d)
                src = [got.get(s, np.zeros(0, dtype=next(iter(got.values())).dtype))
                       for s in range(2 * n1)]
                want = expected(lay, src)
                for s, w in want.items():
                    if not np.array_equal(got[s], w):
                        ok = False
                        print(f"MISMATCH state {name} slot {s}", flush=True)
        g.close()
        if rank == 0:
            print("PASS" if ok else "FAIL", f"world={world} n1={n1} dead={dead}", flush=True)
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    # bench: device time of the pulls, max over ranks
    nb = g.bytes_pulled()
    by_mode = {}
    for mode, ctas in (("interleaved", 0), ("split", 24), ("split", 40), ("split", 64)):
        g.launch_mode, g.peer_ctas = mode, ctas
        times = []
        for it in range(6):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.launch()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if it >= 2:
                times.append(t.item())
        by_mode[f"{mode}{ctas or ''}"] = min(times)
    best = min(by_mode, key=by_mode.get)
    times = [by_mode[best]]
    stats = torch.tensor([nb["local"], nb["peer"]], dtype=torch.float64, device="cuda")
    allb = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(allb, stats)
    if rank == 0:
        ms = min(times)
        per = [b.tolist() for b in allb]
        peer_max = max(p[1] for p in per)
        busiest = max(p[0] + p[1] for p in per)
        print(json.dumps({"workload": f"{shape.name} x{layers} layers, TP{n1} -> comp / TP{n1 - 1} "
                                      f"(rank {dead} of D dead), bf16 param + fp32 master/m/v",
                          "n_gpus": world, "ms": round(ms, 3), "mode": best,
                          "ms_by_mode": {k: round(v, 3) for k, v in by_mode.items()},
                          "bytes_per_gpu_local_peer": per,
                          "busiest_gpu_copy_GBps": round(busiest / ms / 1e6, 1),
                          "busiest_link_GBps": round(peer_max / ms / 1e6, 1)}), flush=True)
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
