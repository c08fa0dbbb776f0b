import time, torch
n = 403440000 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
print("h2d ms", t(lambda: d_a.copy_(h_in, non_blocking=True)))
print("d2h ms", t(lambda: h_out.copy_(d_b, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    s1.synchronize(); s2.synchronize()
print("both ms", t(both))
def chunks(k=16):
    m = n // k
    for i in range(k):
        with torch.cuda.stream(s1): d_a[i*m:(i+1)*m].copy_(h_in[i*m:(i+1)*m], non_blocking=True)
        with torch.cuda.stream(s2): h_out[i*m:(i+1)*m].copy_(d_b[i*m:(i+1)*m], non_blocking=True)
    s1.synchronize(); s2.synchronize()
print("both chunked ms", t(chunks))
import os; print("cpus", os.cpu_count())
