"""Floor of the bench's timing pattern: flush memset, event, replay of a graph holding one
trivial kernel (or three), event.  Diagnostic."""
import torch

s = torch.cuda.Stream()
x = torch.zeros(16, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for nk in (1, 3):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(nk):
            x.add_(1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    for i in range(200):
        with torch.cuda.stream(s):
            fl.zero_()
            ev[i][0].record(s)
            g.replay()
            ev[i][1].record(s)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev[20:])
    print(f"graph with {nk} trivial kernel(s): median {t[len(t) // 2]:.2f} us, min {t[0]:.2f} us")
