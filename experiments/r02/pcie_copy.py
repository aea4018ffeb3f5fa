"""pcie_copy.py — the copy-engine ceiling the end-to-end collect is bound by:
pinned host <-> device copies of the bench's per-step sizes (537 MB of rows
D2H, 8 MB of ids H2D), alone and both directions at once, CUDA events.
    python experiments/r02/pcie_copy.py
"""
import torch


def rate(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return nbytes * reps / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    rows = 1 << 20
    nbytes = rows * 512
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    ids_h = torch.empty(rows * 8, dtype=torch.uint8).pin_memory()
    ids_d = torch.empty(rows * 8, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    print(f"D2H {nbytes >> 20} MB pinned: {rate(lambda: host.copy_(dev, non_blocking=True), nbytes):.1f} GB/s")
    print(f"H2D {nbytes >> 20} MB pinned: {rate(lambda: dev.copy_(host, non_blocking=True), nbytes):.1f} GB/s")
    print(f"H2D {ids_h.numel() >> 20} MB pinned (ids): "
          f"{rate(lambda: ids_d.copy_(ids_h, non_blocking=True), ids_h.numel()):.1f} GB/s")

    def both():
        with torch.cuda.stream(s2):
            dev[: nbytes // 2].copy_(host[: nbytes // 2], non_blocking=True)
        host[nbytes // 2:].copy_(dev[nbytes // 2:], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)

    print(f"H2D + D2H at once ({nbytes >> 21} MB each): {rate(both, nbytes):.1f} GB/s total")


if __name__ == "__main__":
    main()
