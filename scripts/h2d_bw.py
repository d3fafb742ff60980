"""Host-to-device bandwidth from pinned memory (4 GB, 1 / 2 / 4 concurrent copy streams): the e2e
floor of bench.py. Measured on B200: 55.5 GB/s (72 ms per 4 GB) for every split."""
import torch, time
n = 1_000_000_000
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
for ways in (1, 2, 4):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ch = n // ways
        for w in range(ways):
            ss[w].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(ss[w]):
                d[w*ch:(w+1)*ch].copy_(h[w*ch:(w+1)*ch], non_blocking=True)
        for w in range(ways):
            torch.cuda.current_stream().wait_stream(ss[w])
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"ways {ways}: {ms:.2f} ms  {4*n/ms/1e6:.1f} GB/s")
