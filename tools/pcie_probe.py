"""PCIe copy-engine probe: H2D alone, D2H alone, both concurrently (pinned)."""
import time
import torch

n = 16 << 20
for nbytes in (16 << 20, 64 << 20):
    h1 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def t(fn, reps=20):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    def both():
        h2d(); d2h()
    a, b, c = t(h2d), t(d2h), t(both)
    print(f"{nbytes>>20} MiB: H2D {a*1e3:.3f} ms ({nbytes/a/1e9:.1f} GB/s)  D2H {b*1e3:.3f} ms "
          f"({nbytes/b/1e9:.1f} GB/s)  both {c*1e3:.3f} ms (overlap {(a+b)/c:.2f}x)")
