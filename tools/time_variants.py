"""Time k_scale_space-stage variants built with -D experiment flags (performance experiments).
Usage: python tools/time_variants.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
import paper_2108_12050_b200 as mhfd, synth
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * b, dose=300.0, device="cuda") for b in range(8)])
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
for _ in range(2): det.focus_score(imgs)
torch.cuda.synchronize()
det.timing_enable(5)
for _ in range(5): det.focus_score(imgs)
st = det.timing_read()
print(sys.argv[1], "scale_space ms/img %%.4f" %% (sum(s[1] for s in st) / len(st) / 8))
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, MHFD_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, "-c", code, lib], env=env, check=False)
