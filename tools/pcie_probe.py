#!/usr/bin/env python
"""Host<->device copy rates on this box (pinned memory, CUDA events): H2D alone, D2H alone, both
at once on two streams, and H2D split over two streams — the bound of bench.py's e2e step."""
import json
import torch


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both():
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)

    def split():
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d[: n // 2].copy_(h[: n // 2], non_blocking=True)
        with torch.cuda.stream(s2):
            d[n // 2:].copy_(h[n // 2:], non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)

    out = {"h2d_GBps": rate(lambda: d.copy_(h, non_blocking=True), n),
           "d2h_GBps": rate(lambda: h.copy_(d, non_blocking=True), n),
           "h2d_512MB_plus_d2h_256MB_concurrent_ms": 1e3 * (n + n // 2) / 1e9 / rate(both, n + n // 2),
           "h2d_two_streams_GBps": rate(split, n)}
    out["e2e_c3_bound_ms"] = out["h2d_512MB_plus_d2h_256MB_concurrent_ms"]
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
