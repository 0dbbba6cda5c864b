"""Small workload for compute-sanitizer (one tool per gpurun call): the
C1 smoke tile through k_tc<1> (DoG planes) and k_tc<0> (v/argmax) + NMS + k_prune, a
batch of two 1024^2 u8 tiles (k_tc, multi-tile CTAs, 26-neighbour NMS), one 1024^2 u16
tile on the two-pass pair kernels (k_rows_pair / k_cols_pair), single-image bands and
pruning of a gathered list.  Prints the scores; exits non-zero on any CUDA error."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

torch.cuda.set_device(0)
out = []
img = torch.from_numpy(synth.em_tile_np(256, 256, 1000, dose=300.0, bits=8))
det = mhfd.Detector(256, 256, 1.0, 5.0, 5, threshold=0.08, overlap=0.5)
det.debug_dump(img, dog=True, cands=True)
out.append(float(det.focus_score(img)[0]))
imgs = torch.stack([synth.em_tile(1024, 1024, 1000 + b, defocus=1.0 * b, dose=300.0, device="cuda")
                    for b in range(2)])
det2 = mhfd.Detector(1024, 1024, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
out += det2.focus_score(imgs).tolist()
b, c, f = det2.detect(imgs)
det26 = mhfd.Detector(1024, 1024, 1.0, 10.0, 10, threshold=0.09, overlap=0.5, nms="26")
out += det26.focus_score(imgs).tolist()
u16 = synth.em_tile(1024, 1024, 1001, defocus=0.0, dose=300.0, bits=16, device="cuda")
u16 = torch.from_numpy(u16.to(torch.int32).cpu().numpy().astype("uint16")).cuda()
out += det2.focus_score(u16).tolist()
parts, tot = [], 0
for (y0, y1) in ((0, 512), (512, 1024)):
    cc, n = det2.detect_band(imgs[0], y0, y1)
    parts.append(cc[:int(n)].clone())
    tot += int(n)
_, cnt, sc, _ = det2.prune_candidates(torch.cat(parts, 0), tot)
out.append(float(sc[0]))
torch.cuda.synchronize()
print("scores", out)
