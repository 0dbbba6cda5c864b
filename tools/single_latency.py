"""Where does the host-visible latency of ONE 4096^2 u8 tile go (C3, focus_score_host,
chunk 1)?  Prints the pinned H2D copy time alone, the device-resident call, the host call
timed by events on its stream and by the wall clock, the host-side return time of the
call (before the synchronize), and the per-stage device times of the host call."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
img = synth.em_tile(S, S, 1000, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0).contiguous()
host = img.cpu().pin_memory()
det = mhfd.Detector(S, S, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
dst = torch.empty_like(img)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def ev(fn, n=11):
    out = []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(n):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def wall(fn, n=11):
    out, ret = [], []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ret.append((t1 - t0) * 1e3)
        out.append((t2 - t0) * 1e3)
    return statistics.median(out), statistics.median(ret)


print(f"tile {S}^2 u8, {img.numel() / 2**20:.1f} MiB")
print(f"pinned H2D copy alone (events): {ev(lambda: dst.copy_(host, non_blocking=True)):.3f} ms")
print(f"device-resident focus_score (events): {ev(lambda: det.focus_score(img)):.3f} ms")
print(f"focus_score_host chunk 1 (events on stream): {ev(lambda: det.focus_score_host(host, chunk=1)):.3f} ms")
w, r = wall(lambda: det.focus_score_host(host, chunk=1))
print(f"focus_score_host chunk 1 (wall): {w:.3f} ms; call returns after {r:.3f} ms")
w, r = wall(lambda: det.focus_score(img))
print(f"device-resident focus_score (wall): {w:.3f} ms; call returns after {r:.3f} ms")
det.timing_enable(4)
for _ in range(4):
    det.focus_score_host(host, chunk=1)
torch.cuda.synchronize()
for row in det.timing_read():
    print("host-call stages:", " ".join(f"{x:.3f}" for x in row), f"= {sum(row):.3f}")
det.timing_enable(4)
for _ in range(4):
    det.focus_score(img)
torch.cuda.synchronize()
for row in det.timing_read():
    print("device-call stages:", " ".join(f"{x:.3f}" for x in row), f"= {sum(row):.3f}")
