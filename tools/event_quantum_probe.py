import torch
s = torch.cuda.Stream()
torch.cuda._sleep(1000000); torch.cuda.synchronize()
with torch.cuda.stream(s):
    for n in range(100000, 112000, 500):
        ts = []
        for r in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)
            e0.record(s); torch.cuda._sleep(n); e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(n, " ".join(f"{t:.3f}" for t in ts))
