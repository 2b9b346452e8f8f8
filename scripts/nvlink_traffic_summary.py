"""Summarise the ncu CSV of scripts/nvlink_traffic.py into per-GPU NVLink bytes.

    python scripts/nvlink_traffic_summary.py ncu.csv plan.json [algorithmic_bytes]

Takes the last plan-kernel launch on each device (device g ran rank g's plan).
Each kernel's ncu counters are its own GPU's NVLink ports: `nvltx` = what it
wrote to peers (plus its read requests), `nvlrx` = what it read from peers
(plus write acknowledgements); `_data_user` = payload only.  During the real,
concurrent step GPU g also serves the other kernels: it receives their writes
into g and sends the responses to their reads of g.  With two GPUs one link
pair carries everything (GPU 0 TX = kernel 0 TX + kernel 1 RX).  With more,
each kernel's counters are split over its peers in proportion to the bytes its
plan moves to / from each peer (plan.json, from the same plans; at N=2 the
measured user bytes equal the plan's to 1.0003x, so the split is exact to that
level).  Prints per-GPU TX/RX bytes (raw and user data), the busiest direction
and its ratio to the algorithmic bytes.
"""

import csv
import json
import sys


def main():
    path, plan_path = sys.argv[1], sys.argv[2]
    algo = int(sys.argv[3]) if len(sys.argv) > 3 else None
    with open(plan_path) as f:
        plan = json.load(f)
    world = plan["world"]
    per_peer = {int(r): {int(q): v for q, v in d.items()}
                for r, d in plan["read_and_write_bytes_per_peer"].items()}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    kernels = {}
    for r in csv.DictReader(lines):
        if "plan_kernel" not in r.get("Kernel Name", ""):
            continue
        k = kernels.setdefault(r["ID"], {"device": int(r.get("Device", r.get("Device ID", 0))),
                                         "name": r["Kernel Name"][:80]})
        k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    last = {}
    for kid in sorted(kernels, key=int):
        last[kernels[kid]["device"]] = kernels[kid]
    out = {"world": world, "kernels": last}
    for kind, tx_m, rx_m in (("raw", "nvltx__bytes.sum", "nvlrx__bytes.sum"),
                             ("user", "nvltx__bytes_data_user.sum", "nvlrx__bytes_data_user.sum")):
        if not all(tx_m in k for k in last.values()):
            continue
        tx = {g: 0.0 for g in range(world)}
        rx = {g: 0.0 for g in range(world)}
        for j, k in last.items():
            tx[j] += k[tx_m]          # kernel j's own ports
            rx[j] += k[rx_m]
            total = sum(v for q, v in per_peer.get(j, {}).items() if q != j)
            for q, v in per_peer.get(j, {}).items():
                if q == j or total == 0:
                    continue
                rx[q] += k[tx_m] * v / total   # j's writes (and requests) arrive at q
                tx[q] += k[rx_m] * v / total   # q sends j the data j reads
        out[f"per_gpu_{kind}"] = {str(g): {"tx": round(tx[g]), "rx": round(rx[g])} for g in range(world)}
        out[f"busiest_direction_{kind}_bytes"] = round(max(max(tx.values()), max(rx.values())))
    out["busiest_direction_bytes"] = out.get("busiest_direction_raw_bytes")
    out["busiest_direction_user_data_bytes"] = out.get("busiest_direction_user_bytes")
    if algo:
        out["algorithmic_bytes"] = algo
        for kind in ("raw", "user"):
            key = f"busiest_direction_{kind}_bytes"
            if key in out:
                out[f"{kind}_over_algorithmic"] = round(out[key] / algo, 4)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
