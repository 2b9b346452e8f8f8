"""Host link probe for the e2e path: pinned H2D, D2H, and both at once (two
streams), 1 GiB per direction, CUDA events.  Prints JSON."""
import json

import torch


def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def timed(fn, iters=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    res["h2d_GBps"] = round(n / timed(lambda: d_a.copy_(h_in, non_blocking=True)) / 1e6, 1)
    res["d2h_GBps"] = round(n / timed(lambda: h_out.copy_(d_b, non_blocking=True)) / 1e6, 1)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    res["concurrent_per_direction_GBps"] = round(n / timed(both) / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
