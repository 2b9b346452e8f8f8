"""Summarise the ncu CSV of scripts/nvlink_traffic.py into per-GPU NVLink bytes.

    python scripts/nvlink_traffic_summary.py ncu.csv [algorithmic_bytes]

Takes the last plan-kernel launch on each device (device 0 ran rank 0's plan,
device 1 rank 1's) and prints JSON: per kernel its NVLink TX/RX and DRAM
bytes and duration; per GPU the bytes each direction carries during the
concurrent step (own TX + partner RX, own RX + partner TX); and the busiest
direction against the algorithmic bytes (bench roofline.algorithmic_bytes).
"""

import csv
import json
import sys


def main():
    path = sys.argv[1]
    algo = int(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    kernels = {}
    for r in rows:
        if "plan_kernel" not in r.get("Kernel Name", ""):
            continue
        k = kernels.setdefault(r["ID"], {"device": int(r.get("Device", r.get("Device ID", 0))),
                                         "name": r["Kernel Name"][:80]})
        v = float(r["Metric Value"].replace(",", ""))
        k[r["Metric Name"]] = v
    last = {}
    for kid in sorted(kernels, key=int):
        last[kernels[kid]["device"]] = kernels[kid]
    out = {"kernels": last}
    if 0 in last and 1 in last:
        k0, k1 = last[0], last[1]
        g = {
            "gpu0_tx": k0["nvltx__bytes.sum"] + k1["nvlrx__bytes.sum"],
            "gpu0_rx": k0["nvlrx__bytes.sum"] + k1["nvltx__bytes.sum"],
        }
        g["gpu1_tx"], g["gpu1_rx"] = g["gpu0_rx"], g["gpu0_tx"]
        out["per_gpu_direction_bytes"] = g
        busiest = max(g.values())
        out["busiest_direction_bytes"] = busiest
        if "nvltx__bytes_data_user.sum" in k0:
            u = {"gpu0_tx": k0["nvltx__bytes_data_user.sum"] + k1["nvlrx__bytes_data_user.sum"],
                 "gpu0_rx": k0["nvlrx__bytes_data_user.sum"] + k1["nvltx__bytes_data_user.sum"]}
            out["per_gpu_direction_user_data_bytes"] = u
            out["busiest_direction_user_data_bytes"] = max(u.values())
        if algo:
            out["algorithmic_bytes"] = algo
            out["busiest_over_algorithmic"] = round(busiest / algo, 4)
            if "busiest_direction_user_data_bytes" in out:
                out["user_data_over_algorithmic"] = round(
                    out["busiest_direction_user_data_bytes"] / algo, 4)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
