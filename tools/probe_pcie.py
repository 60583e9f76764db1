"""PCIe ceiling for the e2e leg: H2D alone, D2H alone, and both directions
concurrently (pinned host buffers, 134 MB = one C2 X block), GB/s."""
import torch

nbytes = 1 << 27
h = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
d = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d[0].copy_(h[0], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h[1].copy_(d[1], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return reps * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9


run(True, True, 2)
print(f"H2D {run(True, False):.1f} GB/s, D2H {run(False, True):.1f} GB/s, "
      f"both concurrently {run(True, True):.1f} GB/s per direction")
