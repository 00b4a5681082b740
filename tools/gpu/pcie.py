"""PCIe copy rates on the box: pinned H2D / D2H alone and concurrently (separate streams)."""
import torch
n = 176 * 2**20 // 8
h = torch.empty(n, dtype=torch.int64).pin_memory(); d = torch.empty(n, dtype=torch.int64, device="cuda")
h2 = torch.empty(n, dtype=torch.int64).pin_memory(); d2 = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, rep=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(rep): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / rep
def both():
    ev = torch.cuda.Event(); ev.record()
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
GB = n * 8 / 1e9
a = t(lambda: d.copy_(h, non_blocking=True)); b = t(lambda: h2.copy_(d2, non_blocking=True)); c = t(both)
print(f"H2D {GB/a*1e3:.1f} GB/s  D2H {GB/b*1e3:.1f} GB/s  both {2*GB/c*1e3:.1f} GB/s total ({c:.3f} ms vs {a:.3f}+{b:.3f})")
