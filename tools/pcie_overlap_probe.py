import torch, time, threading, json
n = 256 * 1024 * 1024  # 2 GiB of doubles
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    s1.synchronize()
def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s2.synchronize()
def t(fn, reps=3):
    fn(); t0=time.perf_counter()
    for _ in range(reps): fn()
    return (time.perf_counter()-t0)/reps*1e3
def both_one_thread():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s1.synchronize(); s2.synchronize()
def both_threads():
    th=threading.Thread(target=h2d); th.start(); d2h(); th.join()
print(json.dumps({"h2d": t(h2d), "d2h": t(d2h), "both_one_thread": t(both_one_thread), "both_threads": t(both_threads)}))
