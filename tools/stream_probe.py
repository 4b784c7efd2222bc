"""Does a D2H copy on one stream delay work on another stream? (diagnostics)"""
import time
import torch

n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
comp = torch.cuda.current_stream()
down = torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
for variant in ("plain", "record_stream", "event_only"):
    torch.cuda.synchronize()
    base, a0, a1, c0, c1, b0, b1 = E(), E(), E(), E(), E(), E(), E()
    base.record(comp)
    a0.record(comp); torch.cuda._sleep(50_000_000); a1.record(comp)
    ev = torch.cuda.Event(); ev.record(comp)
    with torch.cuda.stream(down):
        down.wait_event(ev)
        c0.record(down)
        if variant != "event_only":
            h.copy_(d, non_blocking=True)
        if variant == "record_stream":
            d.record_stream(down)
        c1.record(down)
    b0.record(comp); torch.cuda._sleep(50_000_000); b1.record(comp)
    torch.cuda.synchronize()
    f = lambda e: base.elapsed_time(e)
    print(variant, f"A {f(a0):.1f}-{f(a1):.1f}  copy {f(c0):.1f}-{f(c1):.1f}  B {f(b0):.1f}-{f(b1):.1f}")
# a small pageable D2H on comp while the big copy runs
torch.cuda.synchronize()
base, c0, c1, b0, b1 = E(), E(), E(), E(), E()
base.record(comp)
with torch.cuda.stream(down):
    c0.record(down); h.copy_(d, non_blocking=True); c1.record(down)
x = torch.ones(4, device="cuda")
b0.record(comp)
t = time.perf_counter(); v = x.sum().item(); dt = time.perf_counter() - t
b1.record(comp)
torch.cuda.synchronize()
print("small .item() during copy:", f"{dt*1e3:.1f} ms host; copy {base.elapsed_time(c0):.1f}-{base.elapsed_time(c1):.1f}")
