"""Which NVML NVLink counters move, and by how much, for a known peer copy?

Copies 4 GiB GPU0 -> GPU1 (one direction) and prints the per-field deltas of
the NVLink throughput / byte counters on both GPUs, per link scope and for the
aggregate scope.  Used to pick the counters bench.py reads for
roofline.traffic at N>1.
"""

from __future__ import annotations

import json
import sys

import pynvml as N
import torch

FIELDS = {138: "THROUGHPUT_DATA_TX(KiB)", 139: "THROUGHPUT_DATA_RX(KiB)",
          140: "THROUGHPUT_RAW_TX(KiB)", 141: "THROUGHPUT_RAW_RX(KiB)",
          202: "COUNT_XMIT_BYTES", 204: "COUNT_RCV_BYTES"}
SCOPES = list(range(18)) + [0xFFFFFFFF]


def read(h):
    out = {}
    for f in FIELDS:
        for s in SCOPES:
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(f, s)])[0]
            except N.NVMLError as e:
                out[(f, s)] = f"err {e}"
                continue
            if v.nvmlReturn != 0:
                out[(f, s)] = f"ret {v.nvmlReturn}"
                continue
            out[(f, s)] = int(v.value.ullVal)
    return out


def main():
    N.nvmlInit()
    hs = [N.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
    nbytes = 4 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0").fill_(1)
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    before = [read(h) for h in hs]
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    after = [read(h) for h in hs]
    res = {"copied_bytes": nbytes, "gpus": []}
    for g in range(2):
        rows = {}
        for key, v0 in before[g].items():
            v1 = after[g][key]
            if isinstance(v0, int) and isinstance(v1, int):
                d = v1 - v0
                if d:
                    rows[f"{FIELDS[key[0]]}@{'all' if key[1] == 0xFFFFFFFF else key[1]}"] = d
            elif key[1] in (0, 0xFFFFFFFF):
                rows[f"{FIELDS[key[0]]}@{'all' if key[1] == 0xFFFFFFFF else key[1]}"] = str(v1)
        res["gpus"].append(rows)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
