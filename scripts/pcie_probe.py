"""Do D2H and H2D copies on different streams overlap on this box? (e2e pipeline check)"""
import time
import torch

n = 160 * 2**20 // 4
dev_a = torch.empty(n, dtype=torch.float32, device="cuda")
dev_b = torch.empty(n, dtype=torch.float32, device="cuda")
host_a = torch.empty(n, dtype=torch.float32, pin_memory=True)
host_b = torch.empty(n, dtype=torch.float32, pin_memory=True)
sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for _ in range(2):
    d2h = t(lambda: host_a.copy_(dev_a, non_blocking=True))
    h2d = t(lambda: dev_b.copy_(host_b, non_blocking=True))

    def both():
        with torch.cuda.stream(sa):
            host_a.copy_(dev_a, non_blocking=True)
        with torch.cuda.stream(sb):
            dev_b.copy_(host_b, non_blocking=True)
    bo = t(both)

    def piped(k=32):
        m = n // k
        evs = []
        with torch.cuda.stream(sa):
            for i in range(k):
                host_a[i * m:(i + 1) * m].copy_(dev_a[i * m:(i + 1) * m], non_blocking=True)
                e = torch.cuda.Event()
                e.record(sa)
                evs.append(e)
        with torch.cuda.stream(sb):
            for i in range(k):
                sb.wait_event(evs[i])
                dev_b[i * m:(i + 1) * m].copy_(host_a[i * m:(i + 1) * m], non_blocking=True)
    pp = t(piped)

    def with_kernel():
        with torch.cuda.stream(sa):
            host_a.copy_(dev_a, non_blocking=True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(sc):
            e0.record(sc)
            x = torch.ones(1, device="cuda")
            e1.record(sc)
        return e0, e1
    torch.cuda.synchronize()
    ta = time.perf_counter()
    e0, e1 = with_kernel()
    e1.synchronize()
    tk = (time.perf_counter() - ta) * 1e3
    print(f"d2h {d2h:.2f} ms ({160/d2h:.1f} GB/s), h2d {h2d:.2f} ms, both {bo:.2f} ms, "
          f"piped round trip {pp:.2f} ms, small kernel on 3rd stream done after {tk:.2f} ms")
