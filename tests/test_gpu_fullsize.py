"""Full-size parity: the CUDA path against the oracle IN FULL at BASELINE.json's sizes,
in the launch configuration bench.py times (north_star tolerances:
responses within 1e-4 of the peak, candidate and kept sets exact outside the ambiguity
band, scores within 1e-3 — Eq. 3).

  * C3/C4 headline: the bench's own 64-tile batch of 4096^2 u8 tiles, one
    mhfd_debug_dump / mhfd_detect_batch / mhfd_focus_score call over all 64 (each
    persistent k_tc CTA walks ~443 tiles); images g = 0 (defocus 0) and g = 32
    (defocus 2.5 px) compared in full (v, argmax, candidates, kept blobs, score), and
    the pruning of every one of the 64 images checked exactly against the oracle's
    greedy rule on the GPU's own candidates.
  * multi-tile path: a batch of 24 1024^2 tiles (1536 k_tc tiles, >= 10 per CTA), every
    image in full.
  * C3 u16: one 4096^2 u16 tile in full (the two-pass schedule).
  * C5 (8192^2 u16, sigma 1-30, 20 scales, R_max 150): v/argmax and candidates on three
    row bands (the top band's blur crosses the periodic wrap, the bottom one ends at
    the image edge) from the oracle's band DoG stack, and the whole image's pruning
    exactly against the oracle on the GPU's candidates.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity as P

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the gpu marker is deselected on CPU runs
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2108_12050_b200 as mhfd  # noqa: E402

C3 = dict(min_sigma=1.0, max_sigma=10.0, num_scales=10)
C5 = dict(min_sigma=1.0, max_sigma=30.0, num_scales=20)
TAU3, TAU5, OVERLAP = 0.09, 0.145, 0.5


def _u16(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.int32).cpu().numpy().astype(np.uint16)


def _image_parity(img_np, cfg, tau, v_g, idx_g, lohi_g, cands_g, kept_g, count_g, score_g, label):
    """Every comparison of the parity procedure for one Eq. 3 image, in full."""
    n = cfg["num_scales"]
    ref = oracle.detect(img_np, cfg["min_sigma"], cfg["max_sigma"], n, tau, OVERLAP, dump=True, grid_prune=True)
    assert tuple(lohi_g) == (ref["lo"], ref["hi"]), (label, lohi_g, ref["lo"], ref["hi"])
    D = ref["D"]
    Pk = float(D.max())
    eps = P.REL_EPS * Pk
    verr = float(np.abs(v_g.astype(np.float64) - ref["v"]).max())
    assert verr <= eps, f"{label}: max |v_gpu - v_oracle| = {verr:.3e} > eps {eps:.3e}"
    tie = P.scale_tie(D, eps)
    del D
    assert np.array_equal(idx_g[~tie], ref["idx"][~tie]), f"{label}: argmax differs outside scale ties"
    amb = P.ambiguous_paper(ref["v"], tau, eps)
    amb_xy = {(int(x), int(y)) for y, x in zip(*np.nonzero(amb))}
    tie_xy = {(int(x), int(y)) for y, x in zip(*np.nonzero(tie))}
    ora_c = P.oracle_rows(oracle.nms_paper_v(ref["v"], ref["idx"], tau))
    summ = P.compare_candidates(cands_g, ora_c, amb_xy, tie_xy, eps, "paper")
    assert cands_g == sorted(cands_g, key=lambda r: (r[1], r[0], r[2]))
    P.assert_prune_exact(cands_g, kept_g, cfg, OVERLAP)
    ora_k = P.oracle_rows(ref["blobs"])
    rad = P.radii(cfg["min_sigma"], cfg["max_sigma"], n)
    pr = P.compare_pruned(kept_g, ora_k, P.pruning_seeds(amb_xy, tie_xy, cands_g, ora_c), max(rad), rad, "paper")
    assert count_g == len(kept_g) and float(score_g) == float(count_g)
    P.assert_score(count_g, ref["count"])
    summ.update(label=label, v_err_rel=verr / Pk, count_gpu=count_g, count_oracle=ref["count"],
                pruned_excluded=pr["excluded"])
    print(summ)
    return summ


def _batch_parity(det, imgs, cfg, tau, check, to_np):
    """One dump / detect / focus_score call over the whole batch (the bench's launch
    configuration); images in `check` compared in full, the pruning of all exactly."""
    B = imgs.shape[0]
    dump = det.debug_dump(imgs, dog=False, cands=True)
    blobs, cnt, flags = det.detect(imgs)
    scores = det.focus_score(imgs)
    torch.cuda.synchronize()
    assert int(flags.max()) == 0
    cnt_h, sc_h, nc_h = cnt.cpu().tolist(), scores.cpu().tolist(), dump["ncand"].cpu().tolist()
    out = []
    for b in range(B):
        cands = P.gpu_rows(dump["cands"][b], min(int(nc_h[b]), det.max_candidates))
        kept = P.gpu_rows(blobs[b], int(cnt_h[b]))
        assert sc_h[b] == float(cnt_h[b])
        if b in check:
            out.append(_image_parity(to_np(imgs[b]), cfg, tau, dump["v"][b].cpu().numpy(),
                                     dump["idx"][b].cpu().numpy(), dump["lohi"][b].tolist(), cands, kept,
                                     int(cnt_h[b]), sc_h[b], f"image {b}"))
        else:
            P.assert_prune_exact(cands, kept, cfg, OVERLAP)
    return out, sc_h


def test_c3_bench_batch_full_parity():
    """The bench's C4 batch (64 x 4096^2 u8, image g: seed 1000+g, defocus 0.5 (g mod 9),
    dose 300) through one call; g = 0 and g = 32 in full, all 64 prunings exact."""
    import bench
    dev = torch.device("cuda", 0)
    imgs = bench.make_batch(0, 64, dev)
    det = mhfd.Detector(4096, 4096, threshold=TAU3, overlap=OVERLAP, **C3)
    assert det.schedule("u8") == "k_tc"
    out, sc = _batch_parity(det, imgs, C3, TAU3, {0, 32}, lambda t: t.cpu().numpy())
    assert out[0]["count_oracle"] > 50000 and out[1]["count_oracle"] > 1000
    assert sc[0] > sc[32]   # defocus 0 vs 2.5 px


def test_c3_dog_planes_full():
    """The DoG planes themselves (Eq. 2, k_tc's plane-writing variant) of one full 4096^2
    tile within 1e-4 of the peak, plane by plane."""
    img = synth.em_tile(4096, 4096, 1000, defocus=0.0, dose=300.0, device="cuda")
    det = mhfd.Detector(4096, 4096, threshold=TAU3, **C3)
    d = det.debug_dump(img, dog=True, cands=False)
    torch.cuda.synchronize()
    a = img.cpu().numpy()
    lo, hi = oracle.percentiles(a)
    D = oracle.dog_stack(oracle.stretch(a, lo, hi), 1.0, 10.0, 10)
    eps = P.REL_EPS * float(D.max())
    for i in range(10):
        err = float(np.abs(d["dog"][0, i].cpu().numpy().astype(np.float64) - D[i]).max())
        assert err <= eps, (i, err, eps)


def test_multitile_batch_1024_full_parity():
    """24 x 1024^2 u8 (1536 k_tc tiles on 148 persistent CTAs: the multi-tile-per-CTA
    path), mixed defocus, every image compared in full."""
    imgs = torch.stack([synth.em_tile(1024, 1024, 2000 + b, defocus=0.25 * (b % 12), dose=300.0, device="cuda")
                        for b in range(24)])
    det = mhfd.Detector(1024, 1024, threshold=TAU3, overlap=OVERLAP, **C3)
    assert det.schedule("u8") == "k_tc"
    out, _ = _batch_parity(det, imgs, C3, TAU3, set(range(24)), lambda t: t.cpu().numpy())
    assert len(out) == 24


def test_c3_u16_full_parity():
    """One 4096^2 u16 tile (sigma 1-10, 10 scales) in full."""
    img = synth.em_tile(4096, 4096, 1000, defocus=0.0, dose=300.0, bits=16, device="cuda")
    img = torch.from_numpy(_u16(img)).cuda().unsqueeze(0)
    det = mhfd.Detector(4096, 4096, threshold=TAU3, overlap=OVERLAP, **C3)
    out, _ = _batch_parity(det, img, C3, TAU3, {0}, lambda t: _u16(t))
    assert out[0]["count_oracle"] > 50000


@pytest.fixture(scope="module")
def c5():
    img = synth.em_tile(8192, 8192, 7, defocus=0.0, dose=300.0, bits=16, device="cuda")
    a = _u16(img)
    det = mhfd.Detector(8192, 8192, threshold=TAU5, overlap=OVERLAP, **C5)
    t = torch.from_numpy(a).cuda()
    dump = det.debug_dump(t, dog=False, cands=True)
    blobs, cnt, flags = det.detect(t)
    scores = det.focus_score(t)
    torch.cuda.synchronize()
    lo, hi = oracle.percentiles(a)
    return {"a": a, "det": det, "dump": dump, "blobs": blobs, "cnt": int(cnt[0]), "flags": int(flags[0]),
            "score": float(scores[0]), "f": oracle.stretch(a, lo, hi), "lohi": (lo, hi)}


@pytest.mark.parametrize("y0,y1", [(0, 256), (4000, 4256), (8064, 8192)])
def test_c5_band_full_parity(c5, y0, y1):
    """C5 rows [y0, y1) in full: v / argmax of the GPU's whole-image run against the
    oracle's DoG stack of rows [y0-1, y1+1) (the blur of the top band reads rows
    -150..: the periodic wrap), and the GPU's candidates in those rows against the
    oracle's Eq. 3 NMS of that stack (-inf padding only at the image edges)."""
    H = 8192
    assert tuple(c5["dump"]["lohi"][0].tolist()) == c5["lohi"]
    r0, r1 = max(0, y0 - 1), min(H, y1 + 1)
    D = oracle.dog_stack(c5["f"], 1.0, 30.0, 20, rows=(r0, r1))
    v, idx = oracle.scale_argmax(D)
    eps = P.REL_EPS * float(D.max())
    vg = c5["dump"]["v"][0, r0:r1].cpu().numpy().astype(np.float64)
    ig = c5["dump"]["idx"][0, r0:r1].cpu().numpy()
    err = float(np.abs(vg - v).max())
    assert err <= eps, (err, eps)
    tie = P.scale_tie(D, eps)
    assert np.array_equal(ig[~tie], idx[~tie])
    # candidates of rows [y0, y1): their 8 neighbours all lie in the stack
    inner = slice(y0 - r0, y1 - r0)
    cand = oracle.nms_paper_v(v, idx, TAU5)
    ora = [(x, y + r0, s, r) for (x, y, s, r) in P.oracle_rows(cand) if y0 <= y + r0 < y1]
    amb = P.ambiguous_paper(v, TAU5, eps)
    amb[:inner.start] = False
    amb[inner.stop:] = False
    amb_xy = {(int(x), int(y) + r0) for y, x in zip(*np.nonzero(amb))}
    tie_xy = {(int(x), int(y) + r0) for y, x in zip(*np.nonzero(tie))}
    nc = int(c5["dump"]["ncand"][0])
    allg = P.gpu_rows(c5["dump"]["cands"][0], min(nc, c5["det"].max_candidates))
    gpu = [r for r in allg if y0 <= r[1] < y1]
    s = P.compare_candidates(gpu, ora, amb_xy, tie_xy, eps, "paper")
    assert s["n_oracle"] > 500
    print(dict(s, rows=(y0, y1), v_err_rel=err / float(D.max())))


def test_c5_pruning_exact_and_score(c5):
    """The whole C5 image: the kept set equals the oracle's greedy pruning of the GPU's
    candidate list exactly, and the score is its size."""
    assert c5["flags"] == 0
    nc = int(c5["dump"]["ncand"][0])
    cands = P.gpu_rows(c5["dump"]["cands"][0], min(nc, c5["det"].max_candidates))
    kept = P.gpu_rows(c5["blobs"][0], c5["cnt"])
    assert len(cands) == nc > 100000
    assert P.assert_prune_exact(cands, kept, C5, OVERLAP) == c5["cnt"] == c5["score"]
