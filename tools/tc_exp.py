"""Time the blur stage (rows a2-a6) of libraries built with -D experiment flags
(performance experiments, results are not meant to be correct).
Usage: python tools/tc_exp.py lib1.so lib2.so ...   (env TC_B = batch, default 16)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, torch
sys.path.insert(0, "%s")
import paper_2108_12050_b200 as mhfd, synth
B = int(os.environ.get("TC_B", "16"))
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b %% 9), dose=300.0, device="cuda") for b in range(B)])
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
for _ in range(2): det.focus_score(imgs)
torch.cuda.synchronize()
det.timing_enable(5)
for _ in range(5): s = det.focus_score(imgs)
st = det.timing_read()
avg = [sum(r[i] for r in st) / len(st) / B for i in range(4)]
print("%%-28s blur ms/img %%.4f  stages %%s  mean score %%.1f" %% (os.path.basename(sys.argv[1]), avg[1], ["%%.4f" %% a for a in avg], float(s.float().mean())))
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, MHFD_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, "-c", code, lib], env=env, check=False)
