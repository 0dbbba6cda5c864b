import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2108_12050_b200 as mhfd, synth
B = 64
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda") for b in range(B)])
host = imgs.cpu().pin_memory()
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for Bc in (8, 16, 64):
    x = imgs[:Bc].contiguous()
    for _ in range(3): det.focus_score(x)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): det.focus_score(x)
    e1.record(); torch.cuda.synchronize()
    print(f"device B={Bc}: {e0.elapsed_time(e1)/5/Bc:.4f} ms/image", flush=True)
# pure H2D bandwidth
d = torch.empty_like(imgs)
torch.cuda.synchronize(); e0.record(); d.copy_(host, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"H2D 1 GiB: {e0.elapsed_time(e1):.2f} ms", flush=True)
for chunk in (8, 16, 32):
    for _ in range(2): det.focus_score_host(host, chunk=chunk)
    torch.cuda.synchronize(); e0.record()
    for _ in range(3): det.focus_score_host(host, chunk=chunk)
    e1.record(); torch.cuda.synchronize()
    print(f"e2e chunk {chunk}: {e0.elapsed_time(e1)/3:.2f} ms/64", flush=True)
