"""Pinned host->device copy rate alone and while the layer step runs (c2 sizes)."""
import sys
import torch

sys.path.insert(0, ".")


def rate(n_bytes, fn, iters=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    return ms, n_bytes / ms / 1e6


def main():
    dev = torch.device("cuda:0")
    n = 196_608_000
    for parts in (1, 5):
        host = [torch.empty(n // parts * 5 // 5, dtype=torch.uint8).pin_memory() for _ in range(parts)]
        devb = [torch.empty_like(h, device=dev) for h in host]
        tot = sum(h.numel() for h in host)

        def cp():
            for h, d in zip(host, devb):
                d.copy_(h, non_blocking=True)
        ms, gbs = rate(tot, cp)
        print(f"H2D {parts} x {tot // parts / 1e6:.0f} MB: {ms:.2f} ms  {gbs:.1f} GB/s")
    host = torch.empty(5 * n, dtype=torch.uint8).pin_memory()
    d = torch.empty_like(host, device=dev)
    ms, gbs = rate(5 * n, lambda: d.copy_(host, non_blocking=True))
    print(f"H2D 1 x {5 * n / 1e6:.0f} MB: {ms:.2f} ms  {gbs:.1f} GB/s")
    # concurrent with an HBM-heavy kernel stream
    side = torch.cuda.Stream()
    x = torch.empty(2 * 1024 ** 3, dtype=torch.uint8, device=dev)

    def both():
        with torch.cuda.stream(side):
            d.copy_(host, non_blocking=True)
        for _ in range(20):
            x.add_(1)
        torch.cuda.current_stream().wait_stream(side)
    ms, gbs = rate(5 * n, both)
    print(f"H2D {5 * n / 1e6:.0f} MB concurrent with 20 x 2 GB add_: {ms:.2f} ms  ({gbs:.1f} GB/s if copy-bound)")
    ms2, _ = rate(1, lambda: [x.add_(1) for _ in range(20)])
    print(f"20 x add_ alone: {ms2:.2f} ms")


if __name__ == "__main__":
    main()
