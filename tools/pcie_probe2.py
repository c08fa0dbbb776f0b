"""PCIe: concurrent H2D + D2H of 403 MB each, whole vs chunked, issue orders and stream priorities."""
import time, torch
n = 403440000 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
for prio in (0, -1):
    s1 = torch.cuda.Stream(priority=prio); s2 = torch.cuda.Stream()
    def chunks(k, order):
        m = n // k
        if order == "interleave":
            for i in range(k):
                with torch.cuda.stream(s1): d_a[i*m:(i+1)*m].copy_(h_in[i*m:(i+1)*m], non_blocking=True)
                with torch.cuda.stream(s2): h_out[i*m:(i+1)*m].copy_(d_b[i*m:(i+1)*m], non_blocking=True)
        else:
            with torch.cuda.stream(s1):
                for i in range(k): d_a[i*m:(i+1)*m].copy_(h_in[i*m:(i+1)*m], non_blocking=True)
            with torch.cuda.stream(s2):
                for i in range(k): h_out[i*m:(i+1)*m].copy_(d_b[i*m:(i+1)*m], non_blocking=True)
        s1.synchronize(); s2.synchronize()
    for k in (1, 4, 8, 16, 32):
        print(f"prio {prio} chunks {k:2d}: interleaved {t(lambda: chunks(k, 'interleave')):.2f} ms, "
              f"grouped {t(lambda: chunks(k, 'grouped')):.2f} ms", flush=True)
