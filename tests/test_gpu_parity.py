"""CUDA path vs oracle, element by element, through the C ABI.

Sizes: C1 (256^2, sigma 1-5, n 5) and C2 (1024^2, sigma 1-10, n 10) in full;
ragged shapes, u16, the minimum image size, degenerate images and every ABI option;
C3/C4-size images (4096^2, the launch configuration bench.py times) on sampled
pixels the oracle evaluates one by one, plus properties.
"""
import math

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

C1 = dict(min_sigma=1.0, max_sigma=5.0, num_scales=5)
C3 = dict(min_sigma=1.0, max_sigma=10.0, num_scales=10)


def _tau(cfg):
    return 0.1 * (cfg["max_sigma"] - cfg["min_sigma"]) / cfg["num_scales"]


def _to_t(img):
    t = torch.from_numpy(np.ascontiguousarray(img))
    return t


def _full_parity(img, cfg, nms="paper", overlap=0.5, strict=False, tau=None, schedule=None, polarity="dark",
                 response="dog", boundary="periodic"):
    """Full comparison on one image: percentiles, DoG stack, v/argmax, candidates,
    pruned blobs, counts and score."""
    H, W = img.shape
    tau = _tau(cfg) if tau is None else tau
    n = cfg["num_scales"]
    det = mhfd.Detector(W, H, threshold=tau, overlap=overlap, nms=nms, strict=strict, schedule=schedule,
                        polarity=polarity, response=response, boundary=boundary, **cfg)
    dump = det.debug_dump(_to_t(img))
    ref = oracle.detect(img, cfg["min_sigma"], cfg["max_sigma"], n, tau, overlap, nms=nms, strict=strict, dump=True,
                        polarity=polarity, response=response, boundary=boundary)
    # a1: percentiles, exact integers
    lo, hi = dump["lohi"][0].tolist()
    if img.dtype == np.float32:   # float32 bit patterns (reading R24)
        lo, hi = lo & 0xFFFFFFFF, hi & 0xFFFFFFFF
    assert (lo, hi) == (ref["lo"], ref["hi"])
    # a2-a5: responses within 1e-4 of the peak
    D = ref["D"]
    Pk = float(D.max())
    eps = P.REL_EPS * max(Pk, 1e-30)
    Dg = dump["dog"][0].cpu().numpy().astype(np.float64)
    err = float(np.abs(Dg - D).max())
    assert err <= eps, f"max |DoG_gpu - DoG_oracle| = {err:.3e} > eps = {eps:.3e} (P = {Pk:.4f})"
    # a6: inner argmax
    tie = P.scale_tie(D, eps)
    if nms == "paper":
        vg = dump["v"][0].cpu().numpy().astype(np.float64)
        assert float(np.abs(vg - ref["v"]).max()) <= eps
        ig = dump["idx"][0].cpu().numpy()
        assert np.array_equal(ig[~tie], ref["idx"][~tie])
        amb = P.ambiguous_paper(ref["v"], tau, eps)
        amb_xy = {(int(x), int(y)) for y, x in zip(*np.nonzero(amb))}
        ora_c = P.oracle_rows(oracle.nms_paper(D, tau, strict))
    else:
        amb = P.ambiguous_26(D, tau, eps)
        amb_xy = {(int(x), int(y), int(i)) for i, y, x in zip(*np.nonzero(amb))}
        ora_c = P.oracle_rows(oracle.nms_26(D, tau, strict))
    tie_xy = {(int(x), int(y)) for y, x in zip(*np.nonzero(tie))}
    # a7-a8: candidates (ordered list)
    nc = int(dump["ncand"][0])
    gpu_c = P.gpu_rows(dump["cands"][0], min(nc, det.max_candidates))
    assert gpu_c == sorted(gpu_c, key=lambda r: (r[1], r[0], r[2])), "candidate list not in (y, x, scale) order"
    summ = P.compare_candidates(gpu_c, ora_c, amb_xy, tie_xy, eps, nms)
    if nms == "paper" and img.dtype == np.uint8:
        # the fused u8 schedule detect/focus_score run (k_tc when the tile fits, else
        # k_band): v, argmax and candidates without the DoG dump
        fused = det.debug_dump(_to_t(img), dog=False, cands=True)
        vf = fused["v"][0].cpu().numpy().astype(np.float64)
        assert float(np.abs(vf - ref["v"]).max()) <= eps, (det.schedule(), float(np.abs(vf - ref["v"]).max()), eps)
        iff = fused["idx"][0].cpu().numpy()
        assert np.array_equal(iff[~tie], ref["idx"][~tie]), det.schedule()
        ncf = int(fused["ncand"][0])
        gpu_cf = P.gpu_rows(fused["cands"][0], min(ncf, det.max_candidates))
        P.compare_candidates(gpu_cf, ora_c, amb_xy, tie_xy, eps, nms)
        summ["fused_v_err_rel"] = float(np.abs(vf - ref["v"]).max()) / max(Pk, 1e-30)
    # a9-a10: pruned blobs, counts, score
    blobs, cnt, flags = det.detect(_to_t(img))
    scores = det.focus_score(_to_t(img))
    torch.cuda.synchronize()
    count = int(cnt[0])
    assert int(flags[0]) == 0
    assert float(scores[0]) == float(count)
    gpu_k = P.gpu_rows(blobs[0], count)
    assert gpu_k == sorted(gpu_k, key=lambda r: (r[1], r[0], r[2]))
    ora_k = P.oracle_rows(ref["blobs"])
    amb_pts = (P.pruning_seeds(amb_xy, tie_xy, gpu_c, ora_c) if nms == "paper"
               else [(x, y) for (x, y, *_) in ([(k[0], k[1]) for k in amb_xy])])
    rad = P.radii(cfg["min_sigma"], cfg["max_sigma"], n)
    P.compare_pruned(gpu_k, ora_k, amb_pts, max(rad), rad, nms)
    P.assert_score(count, ref["count"])
    summ.update(count_gpu=count, count_oracle=ref["count"], dog_err_rel=err / max(Pk, 1e-30))
    return summ


@pytest.fixture(scope="module")
def c1_img():
    return synth.em_tile_np(256, 256, 1000, dose=300.0, bits=8)


@pytest.mark.parametrize("nms", ["paper", "26"])
@pytest.mark.parametrize("overlap", [0.5, 1.0, 0.0])
def test_c1_full_parity(c1_img, nms, overlap):
    s = _full_parity(c1_img, C1, nms=nms, overlap=overlap)
    assert s["n_oracle"] > 100


@pytest.mark.parametrize("strict", [True])
def test_c1_strict(c1_img, strict):
    _full_parity(c1_img, C1, strict=strict)


@pytest.mark.parametrize("defocus", [0.0, 2.0])
@pytest.mark.parametrize("bits", [8, 16])
def test_c2_pair_parity(defocus, bits):
    img = synth.em_tile_np(1024, 1024, 1000, defocus=defocus, dose=300.0, bits=bits)
    _full_parity(img, C3)


@pytest.mark.parametrize("schedule", ["band", "generic"])
def test_c2_cuda_core_schedules(schedule):
    """The CUDA-core schedules (selectable fallbacks of k_tc) against the oracle."""
    img = synth.em_tile_np(1024, 1024, 1000, defocus=0.0, dose=300.0, bits=8)
    det = mhfd.Detector(1024, 1024, threshold=0.09, schedule=schedule, **C3)
    assert det.schedule("u8") == {"band": "k_band", "generic": "k_scale_space"}[schedule]
    _full_parity(img, C3, schedule=schedule)


@pytest.mark.parametrize("nms,bits,size", [("paper", 8, 256), ("paper", 8, 1024), ("26", 8, 256), ("paper", 16, 256),
                                           ("26", 16, 256)])
def test_bright_polarity_parity(nms, bits, size):
    """Bright features (negated Eq. 2) on every schedule kind: k_tc (u8),
    26-mode and u16 (generic)."""
    img = synth.em_tile_np(size, size, 1002, dose=300.0, bits=bits)
    cfg = C1 if size == 256 else C3
    s = _full_parity(img, cfg, nms=nms, polarity="bright")
    assert s["n_oracle"] > 50


def test_u8_schedule_is_tensor_core():
    """The bench configuration (4096^2 u8, sigma 1-10, n 10) and C2 run the tcgen05 kernel."""
    assert mhfd.Detector(4096, 4096, threshold=0.09, **C3).schedule("u8") == "k_tc"
    assert mhfd.Detector(1024, 1024, threshold=0.09, **C3).schedule("u8") == "k_tc"
    assert mhfd.Detector(256, 256, threshold=0.08, **C1).schedule("u8") == "k_tc"
    assert mhfd.Detector(1024, 1024, threshold=0.09, **C3).schedule("u16") == "k_tc2"
    assert mhfd.Detector(1024, 1024, threshold=0.09, **C3).schedule("f32") == "k_tc2"
    assert mhfd.Detector(1024, 1024, 1.0, 20.0, 12, threshold=0.16).schedule("u8") == "k_tc2"   # R 100 > k_tc's tile
    assert mhfd.Detector(1024, 1024, threshold=0.09, schedule="band", **C3).schedule("u16") == "k_rows_pair+k_cols_pair"
    assert mhfd.Detector(1000, 1000, threshold=0.09, **C3).schedule("u16") == "k_scale_space"   # W % 128 != 0


def test_u16_generic_schedule_parity():
    """The fused generic kernel (k_scale_space: u16 with MHFD_SCHEDULE=generic, widths that
    are not multiples of 256, DoG dumps below R_max 96) against the oracle."""
    img = synth.em_tile_np(1024, 1024, 1004, defocus=1.0, dose=300.0, bits=16)
    det = mhfd.Detector(1024, 1024, threshold=0.09, schedule="generic", **C3)
    assert det.schedule("u16") == "k_scale_space"
    _full_parity(img, C3, schedule="generic")


def test_c2_sharp_beats_defocused():
    imgs = np.stack([synth.em_tile_np(1024, 1024, 1000, defocus=s, dose=300.0) for s in (0.0, 2.0)])
    det = mhfd.Detector(1024, 1024, threshold=0.09, **C3)
    sc = det.focus_score(torch.from_numpy(imgs)).cpu().tolist()
    assert sc[0] > sc[1] > 0


@pytest.mark.parametrize("shape,bits", [((257, 300), 8), ((300, 257), 16), ((51, 51), 8), ((77, 130), 16),
                                        ((200, 1100), 8), ((1030, 250), 8), ((700, 1000), 8)])
def test_ragged_and_minimum_shapes(shape, bits):
    H, W = shape
    img = synth.em_tile_np(H, W, 42, dose=300.0, bits=bits)
    _full_parity(img, C1)


def test_degenerate_and_constant():
    img = synth.constant_image(128, 96, 200)
    det = mhfd.Detector(96, 128, threshold=0.08, **C1)
    blobs, cnt, flags = det.detect(_to_t(img))
    assert int(cnt[0]) == 0
    d = det.debug_dump(_to_t(img))
    assert d["lohi"][0].tolist() == [200, 200]
    assert float(d["dog"].abs().max()) == 0.0


def test_batch_invariance_and_determinism():
    imgs = np.stack([synth.em_tile_np(256, 320, 1000 + b, dose=300.0) for b in range(5)])
    imgs[3] = 77  # a degenerate image inside the batch
    det = mhfd.Detector(320, 256, threshold=0.08, **C1)
    b_all, c_all, _ = det.detect(torch.from_numpy(imgs))
    b_again, c_again, _ = det.detect(torch.from_numpy(imgs))
    assert torch.equal(c_all, c_again)
    for b in range(5):
        k = int(c_all[b])
        assert torch.equal(b_all[b, :k], b_again[b, :k])
    for b in range(5):
        b1, c1, _ = det.detect(torch.from_numpy(imgs[b:b + 1]))
        assert int(c1[0]) == int(c_all[b])
        k = int(c1[0])
        assert torch.equal(b1[0, :k], b_all[b, :k])
    assert int(c_all[3]) == 0


def test_capacity_truncation_and_flags(c1_img):
    det = mhfd.Detector(256, 256, threshold=0.08, **C1)
    full, cnt, fl = det.detect(_to_t(c1_img))
    k = int(cnt[0])
    small, cnt2, fl2 = det.detect(_to_t(c1_img), blob_capacity=17)
    assert int(cnt2[0]) == k and int(fl2[0]) == 2 and int(fl[0]) == 0
    assert torch.equal(small[0, :17], full[0, :17])
    det2 = mhfd.Detector(256, 256, threshold=0.08, max_candidates=50, **C1)
    _, cnt3, fl3 = det2.detect(_to_t(c1_img))
    assert int(fl3[0]) & 1


def test_isolated_disk_gpu():
    img = synth.disk_image(112, 112, 56.5, 56.5, 6.0, contrast=0.6, bits=16)
    det = mhfd.Detector(112, 112, threshold=0.09, **C3)
    blobs, cnt, _ = det.detect(_to_t(img))
    rows = P.gpu_rows(blobs[0], int(cnt[0]))
    ref = oracle.detect(img, 1.0, 10.0, 10, 0.09, 0.5)
    assert [(r[0], r[1], r[2]) for r in rows] == [(56, 56, int(ref["blobs"][0]["scale"]))]


def test_abi_errors_on_gpu():
    det = mhfd.Detector(256, 256, **C1)
    bad = torch.zeros((1, 255, 256), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        det.focus_score(bad)
    with pytest.raises(mhfd.MHFDError):
        mhfd.Detector(40, 40, **C1)   # smaller than 2*ceil(5*max_sigma)+1


# ------------------------------------------------------------------ full size (4096^2)
@pytest.fixture(scope="module")
def c3_batch():
    # generated on the GPU (fast); the oracle gets the same bytes
    imgs = [synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * b, dose=300.0, device="cuda") for b in range(3)]
    return torch.stack(imgs)


def test_c3_sampled_pixels_and_properties(c3_batch):
    """Bench launch configuration (4096^2, sigma 1-10, n 10): sampled responses vs the
    oracle's per-pixel 2-D definition, Eq. 3 decisions at those pixels, properties."""
    B = c3_batch.shape[0]
    det = mhfd.Detector(4096, 4096, threshold=0.09, **C3)
    dump = det.debug_dump(c3_batch, dog=False, cands=True)
    blobs, cnt, flags = det.detect(c3_batch)
    scores = det.focus_score(c3_batch)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    for b in range(B):
        img = c3_batch[b].cpu().numpy()
        lo, hi = oracle.percentiles(img)
        assert dump["lohi"][b].tolist() == [lo, hi]
        f = oracle.stretch(img, lo, hi)
        v = dump["v"][b].cpu().numpy()
        idx = dump["idx"][b].cpu().numpy()
        pts = [(int(y), int(x)) for y, x in rng.integers(0, 4096, size=(12, 2))]
        pts += [(0, 0), (4095, 4095), (0, 4095), (2048, 31), (2048, 32)]
        peak = 0.0
        vals = {}
        for (y, x) in pts:
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    yy, xx = (y + dy) % 4096, (x + dx) % 4096
                    if (yy, xx) not in vals:
                        vals[(yy, xx)] = oracle.dog_at(f, 1.0, 10.0, 10, yy, xx)
                        peak = max(peak, float(vals[(yy, xx)].max()))
        eps = P.REL_EPS * max(peak, 0.05)
        for (yy, xx), Dv in vals.items():
            assert abs(float(v[yy, xx]) - Dv.max()) <= eps
            s = np.sort(Dv)
            if s[-1] - s[-2] > eps:
                assert int(idx[yy, xx]) == int(np.argmax(Dv))
        # Eq. 3 decision at the sampled interior pixels
        cand_set = {(r[0], r[1]) for r in P.gpu_rows(dump["cands"][b], min(int(dump["ncand"][b]), det.max_candidates))}
        for (y, x) in pts:
            if not (1 <= y < 4095 and 1 <= x < 4095):
                continue
            c = vals[(y, x)].max()
            m = max(vals[((y + dy) % 4096, (x + dx) % 4096)].max() for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                    if dy or dx)
            if abs(c - m) > eps and abs(c - 0.09) > eps:
                assert ((x, y) in cand_set) == (c >= m and c > 0.09)
        # properties of the outputs
        k = int(cnt[b])
        assert float(scores[b]) == float(k) and int(flags[b]) == 0 and k > 0
        rows = P.gpu_rows(blobs[b], k)
        assert rows == sorted(rows, key=lambda r: (r[1], r[0], r[2]))
        assert all(r[3] > 0.09 for r in rows)
    sc = scores.cpu().tolist()
    assert sc[0] > sc[1] > sc[2], sc   # defocus 0, 0.5, 1.0 px


# ------------------------------------------------------------------ C5: 8192^2 u16, sigma 1-30, 20 scales
def test_c5_large_radius_sampled():
    """Large-kernel-radius stress (config C5): R up to 150 takes the generic schedule;
    sampled pixels vs the oracle's 2-D definition, argmax, properties."""
    img = synth.em_tile(8192, 8192, 7, defocus=0.0, dose=300.0, bits=16, device="cuda")
    img16 = img.to(torch.int32).cpu().numpy().astype(np.uint16)
    t16 = torch.from_numpy(img16)
    C5 = dict(min_sigma=1.0, max_sigma=30.0, num_scales=20)
    det = mhfd.Detector(8192, 8192, threshold=0.145, **C5)
    dump = det.debug_dump(t16, dog=False, cands=False)
    scores, cnt = det.focus_score(t16, counts=True)
    torch.cuda.synchronize()
    lo, hi = oracle.percentiles(img16)
    assert dump["lohi"][0].tolist() == [lo, hi]
    f = oracle.stretch(img16, lo, hi)
    v = dump["v"][0].cpu().numpy()
    idx = dump["idx"][0].cpu().numpy()
    rng = np.random.default_rng(11)
    pts = [(int(y), int(x)) for y, x in rng.integers(0, 8192, size=(24, 2))] + [(0, 0), (8191, 8191), (4096, 127)]
    vals = {p: oracle.dog_at(f, 1.0, 30.0, 20, p[0], p[1]) for p in pts}
    peak = max(float(d.max()) for d in vals.values())
    eps = P.REL_EPS * max(peak, 0.1)
    for (y, x), Dv in vals.items():
        assert abs(float(v[y, x]) - Dv.max()) <= eps, ((y, x), float(v[y, x]), Dv.max(), eps)
        s = np.sort(Dv)
        if s[-1] - s[-2] > eps:
            assert int(idx[y, x]) == int(np.argmax(Dv))
    assert int(cnt[0]) > 0 and float(scores[0]) == float(int(cnt[0]))


def test_c2_26_mode_parity():
    img = synth.em_tile_np(1024, 1024, 1000, defocus=0.0, dose=300.0, bits=8)
    _full_parity(img, C3, nms="26")


@pytest.mark.parametrize("strict,polarity,tau", [(False, "dark", 1e-6), (True, "bright", None)])
def test_26_mode_row_kernel_parity(strict, polarity, tau):
    """k_nms26_roll (26-neighbour count + park over whole 1024-pixel row segments) and
    k_nms_gather4<26>: full parity at 1024^2 with a threshold low enough that many
    segments overflow their 64-record slabs (re-evaluated in (x, scale) order), and with
    the strict rule and bright polarity."""
    img = synth.em_tile_np(1024, 1024, 1010, defocus=0.5, dose=300.0, bits=8)
    s = _full_parity(img, C3, nms="26", strict=strict, polarity=polarity, tau=tau)
    assert s["n_oracle"] > 1000
    if tau is not None:   # the overflow path was taken: some row segment has > 64 candidates
        det = mhfd.Detector(1024, 1024, threshold=tau, nms="26", strict=strict, polarity=polarity, **C3)
        d = det.debug_dump(_to_t(img), dog=False, cands=True)
        nc = int(d["ncand"][0])
        c = d["cands"][0][:nc].cpu().numpy()
        per_seg = np.bincount(c[:, 1].astype(np.int64) * 1 + (c[:, 0].astype(np.int64) // 1024), minlength=1024)
        assert int(per_seg.max()) > 64, int(per_seg.max())


def test_26_mode_batch_matches_single():
    """26 mode on a batch of two 2048^2 tiles (two segments per row, image index in the
    slab and offset arrays): the same kept blobs as two single-image calls."""
    imgs = np.stack([synth.em_tile_np(2048, 2048, 1020 + k, defocus=1.0 * k, dose=300.0, bits=8) for k in range(2)])
    det = mhfd.Detector(2048, 2048, threshold=_tau(C3), nms="26", **C3)
    t = torch.from_numpy(imgs).cuda()
    blobs, cnt, _ = det.detect(t)
    torch.cuda.synchronize()
    for k in range(2):
        b1, c1, _ = det.detect(t[k:k + 1])
        torch.cuda.synchronize()
        n = int(c1[0])
        assert n > 1000 and n == int(cnt[k]) and torch.equal(b1[0, :n], blobs[k, :n])


# ------------------------------------------------------------------ f2: single-image bands
@pytest.mark.parametrize("size,G", [(1024, 1), (1024, 3), (4096, 2), (4096, 8)])
def test_band_sharding_matches_whole_image(size, G):
    """Single-image multi-GPU sharding, the G ranks run one after
    another on this GPU: the bands' candidate lists (mhfd_detect_band) concatenated in
    band order are bit-identical to the whole image's list, and pruning them
    (mhfd_prune_candidates) reproduces detect()/focus_score() exactly."""
    from paper_2108_12050_b200.dist import band_rows
    img = synth.em_tile(size, size, 1004, defocus=0.5, dose=300.0, device="cuda")
    det = mhfd.Detector(size, size, threshold=0.09, **C3)
    full = det.debug_dump(img, dog=False, cands=True)
    nfull = int(full["ncand"][0])
    blobs_full, cnt_full, _ = det.detect(img)
    score_full = det.focus_score(img)
    parts, total = [], 0
    for r in range(G):
        y0, y1 = band_rows(size, G, r)
        c, n = det.detect_band(img, y0, y1)
        n = int(n)
        parts.append(c[:n].clone())
        total += n
    allc = torch.cat(parts, 0)
    assert total == nfull
    assert torch.equal(allc, full["cands"][0, :nfull])
    blobs, cnt, score, flags = det.prune_candidates(allc, total)
    torch.cuda.synchronize()
    k = int(cnt[0])
    assert k == int(cnt_full[0]) and float(score[0]) == float(score_full[0]) == float(k) and int(flags[0]) == 0
    assert torch.equal(blobs[:k], blobs_full[0, :k])


@pytest.mark.parametrize("G", [1, 3, 8])
def test_band_sharding_pair_schedule_u16(G):
    """Single-image bands on the two-pass pair schedule (u16, sigma 1-20, R_max = 100; the
    f2 case the paper targets: wide scale ranges at full resolution): each band computes
    only the Rx rows and 256-row output tiles its rows need (with the periodic wrap for
    the first and last band), and the concatenated candidate lists equal the whole-image
    list bit for bit; pruning them reproduces detect() exactly."""
    from paper_2108_12050_b200.dist import band_rows
    size = 1024
    a = synth.em_tile_np(size, size, 1009, defocus=0.5, dose=300.0, bits=16)
    img = torch.from_numpy(a.astype(np.int32)).cuda().to(torch.uint16)
    det = mhfd.Detector(size, size, 1.0, 20.0, 12, threshold=0.1 * 19.0 / 12)
    assert det.schedule("u16") == "k_tc2"
    full = det.debug_dump(img, dog=False, cands=True)
    nfull = int(full["ncand"][0])
    blobs_full, cnt_full, _ = det.detect(img)
    parts, total = [], 0
    for r in range(G):
        y0, y1 = band_rows(size, G, r)
        c, n = det.detect_band(img, y0, y1)
        n = int(n)
        parts.append(c[:n].clone())
        total += n
    allc = torch.cat(parts, 0)
    assert total == nfull
    assert torch.equal(allc, full["cands"][0, :nfull])
    blobs, cnt, score, flags = det.prune_candidates(allc, total)
    torch.cuda.synchronize()
    k = int(cnt[0])
    assert k == int(cnt_full[0]) and torch.equal(blobs[:k], blobs_full[0, :k])


# ------------------------------------------------------------------ large radii: two-pass schedule
def test_twopass_matches_fused_generic_bitwise():
    """The two-pass large-radius schedule (k_rows2 / k_cols2) computes the same f32 sums
    as the fused generic kernel: v, argmax, DoG planes, candidates and kept blobs are
    bit-identical (u16, sigma 1-20, R_max = 100)."""
    import os
    img = synth.em_tile(1024, 1024, 1005, defocus=0.0, dose=300.0, bits=16, device="cuda")
    img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16))
    cfg = dict(min_sigma=1.0, max_sigma=20.0, num_scales=12)
    outs = []
    os.environ["MHFD_NO_COLS_PAIR"] = "1"   # paper mode on k_rows2 / k_cols_all, not the pair kernels
    try:
        for flag in (None, "1"):
            if flag:
                os.environ["MHFD_NO_TWOPASS"] = flag
            try:   # "band": the CUDA-core schedules (no tensor-core kernel takes the u16 image)
                det = mhfd.Detector(1024, 1024, threshold=0.1 * 19.0 / 12, schedule="band", **cfg)
            finally:
                os.environ.pop("MHFD_NO_TWOPASS", None)
            assert det.schedule("u16") == ("k_rows2+k_cols_all" if flag is None else "k_scale_space")
            d = det.debug_dump(img, dog=True, cands=True)
            blobs, cnt, _ = det.detect(img)
            torch.cuda.synchronize()
            outs.append((d, blobs, int(cnt[0])))
    finally:
        os.environ.pop("MHFD_NO_COLS_PAIR", None)
    (a, ba, ka), (b, bb, kb) = outs
    for key in ("lohi", "dog", "v", "idx", "ncand"):
        assert torch.equal(a[key], b[key]), key
    n = int(a["ncand"][0])
    assert torch.equal(a["cands"][0, :n], b["cands"][0, :n])
    assert ka == kb > 0 and torch.equal(ba[0, :ka], bb[0, :kb])


def test_cols_pair_matches_cols_all():
    """k_rows_pair + k_cols_pair (paper-mode passes of the two-pass schedule: tap-order
    sums, 8x2 pixels per thread) against k_rows2 + k_cols_all (conv4_row / conv8_col):
    the same f32 taps, so v agrees to a few ulp of the level sums; the argmax agrees except
    at near-ties; the kept blob count agrees within a few near-threshold blobs.  Ragged
    last band (H = 1000) and a degenerate (constant) image in the batch."""
    import os
    imgs = [synth.em_tile(1000, 1024, 1105 + k, defocus=0.5 * k, dose=300.0, bits=16, device="cuda") for k in range(2)]
    imgs.append(torch.full((1000, 1024), 777, dtype=torch.int32))
    img = torch.from_numpy(np.stack([t.to(torch.int32).cpu().numpy() for t in imgs]).astype(np.uint16))
    det = mhfd.Detector(1024, 1000, min_sigma=1.0, max_sigma=20.0, num_scales=12, threshold=0.1 * 19.0 / 12,
                        schedule="band")
    assert det.schedule("u16") == "k_rows_pair+k_cols_pair"
    res = []
    for flag in (None, "1"):
        if flag:
            os.environ["MHFD_NO_COLS_PAIR"] = flag
        try:
            d = det.debug_dump(img, dog=False, cands=False)
            blobs, cnt, _ = det.detect(img)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("MHFD_NO_COLS_PAIR", None)
        res.append((d["v"].cpu(), d["idx"].cpu(), cnt.cpu()))
    (va, ia, ca), (vb, ib, cb) = res
    scale = float(vb.abs().max())
    diff = float((va - vb).abs().max())
    mism = float((ia != ib).float().mean())
    print(f"cols_pair: max|dv| {diff:.3e} (max|v| {scale:.3e}), argmax mismatch {mism:.2e}, counts {ca.tolist()} {cb.tolist()}")
    # both sides sum the same 2R+1 <= 201 f32 products per pass (|x| <= 1 normalised,
    # taps summing to 1), each pass within (2R+1) u of the exact sum, and the column pass
    # carries the row pass's error through taps summing to 1; the DoG scales the
    # difference of two levels by t_i <= 20: |dv| <= 20 * 2 * 2 * 201 * 2^-24 = 9.6e-4
    # (worst case); typical errors are random-walk sized, so the mean is held far lower
    assert diff <= 9.6e-4, (diff, scale)
    assert float((va - vb).abs().mean()) <= 1e-6
    assert mism < 1e-3
    assert float(va[2].abs().max()) == 0.0 and int(ia[2].max()) == 0 and int(ca[2]) == 0
    for k in range(2):
        assert abs(int(ca[k]) - int(cb[k])) <= max(2, int(cb[k]) // 500), (k, int(ca[k]), int(cb[k]))


def test_nms_dense_candidates_exact():
    """Dense local maxima (uniform noise, tiny threshold): most 1024-pixel segments hold
    more candidates than their count-pass slab (32), so the gather re-evaluates them.  The
    candidate list must equal the oracle's Eq. 3 NMS applied to the GPU's own v (same f32
    values, so the comparison is exact), in raster order, with the GPU's argmax."""
    rng = np.random.default_rng(17)
    img = rng.integers(0, 256, size=(1024, 1024), dtype=np.uint8)
    det = mhfd.Detector(1024, 1024, min_sigma=1.0, max_sigma=3.0, num_scales=2, threshold=1e-6, overlap=1.0)
    d = det.debug_dump(_to_t(img), dog=False, cands=True)
    torch.cuda.synchronize()
    v = d["v"][0].cpu().numpy().astype(np.float64)
    ref = oracle.nms_paper(v[None], 1e-6)
    n = int(d["ncand"][0])
    assert n == len(ref) and n > 32 * 1024   # > 32 per segment on average
    got = d["cands"][0, :n].cpu()
    np.testing.assert_array_equal(got[:, 0].numpy(), ref["x"])
    np.testing.assert_array_equal(got[:, 1].numpy(), ref["y"])
    idx = d["idx"][0].cpu().numpy()
    np.testing.assert_array_equal(got[:, 2].numpy(), idx[ref["y"], ref["x"]])
    np.testing.assert_array_equal(got[:, 3].view(torch.float32).numpy().astype(np.float64), ref["response"])


def test_defocus_sweep_log_linear():
    """the focus score falls log-linearly with defocus (the paper fits
    r = -0.9754 on a real focal series).  Synthetic 1024^2 sweep 0..4 px at dose 300:
    counts strictly decrease and the log-linear fit has r <= -0.95 (advisory bound, the
    survey measured -0.986 on this generator)."""
    from paper_2108_12050_b200.calibrate import fit_log_linear
    defocus = np.arange(0.0, 4.01, 0.5)
    imgs = torch.stack([synth.em_tile(1024, 1024, 1000, defocus=float(s), dose=300.0, device="cuda") for s in defocus])
    det = mhfd.Detector(1024, 1024, threshold=0.09, **C3)
    scores = det.focus_score(imgs).cpu().numpy()
    assert np.all(np.diff(scores) < 0), scores
    fit = fit_log_linear(defocus, scores)
    assert fit.r <= -0.95 and fit.slope < 0, fit
    np.testing.assert_allclose(fit.deviation(fit.predict(defocus)), defocus, atol=1e-9)


@pytest.mark.parametrize("dtype", [torch.uint8, torch.uint16])
def test_downsample_bit_exact(dtype):
    """mhfd_downsample (f4 pre-step) vs the oracle's f64 bilinear: integer outputs,
    bit-exact, on ragged shapes, factors 1-5 and 8, a batch of 3 (each image vs its own
    oracle call); then the downsampled tile feeds the detector."""
    rng = np.random.default_rng(77)
    hi = 256 if dtype == torch.uint8 else 65536
    npd = np.uint8 if dtype == torch.uint8 else np.uint16
    for (H, W) in ((1000, 777), (64, 64), (257, 1031), (255, 128)):   # (64, 64), (255, 128): factor-2 fast path
        a = rng.integers(0, hi, size=(3, H, W)).astype(npd)
        t = torch.from_numpy(a.astype(np.int32)).to(torch.int32).cuda().to(dtype) if dtype == torch.uint16 \
            else torch.from_numpy(a).cuda()
        for f in (1, 2, 3, 4, 5, 8):
            out = mhfd.downsample(t, f)
            torch.cuda.synchronize()
            assert out.shape == (3, -(-H // f), -(-W // f)) and out.dtype == dtype
            o = out.cpu()
            o = o.numpy() if dtype == torch.uint8 else o.to(torch.int32).numpy().astype(np.uint16)
            for b in range(3):
                assert np.array_equal(o[b], oracle.downsample(a[b], f)), (H, W, f, b)
    with pytest.raises(mhfd.MHFDError):
        mhfd.downsample(torch.zeros((1, 8, 8), dtype=dtype, device="cuda"), 9)
    # the pre-step in front of the detector: a 2048^2 synthetic tile -> 1024^2
    img = synth.em_tile(2048, 2048, 1000, defocus=0.0, dose=300.0, device="cuda")
    if dtype == torch.uint8:
        small = mhfd.downsample(img, 2)[0]
        det = mhfd.Detector(1024, 1024, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
        s = float(det.focus_score(small)[0])
        ref = oracle.detect(small.cpu().numpy(), 1.0, 10.0, 10, 0.09, 0.5)["count"]
        assert abs(s - ref) <= 1e-3 * ref


# ---------------------------------------------------------------- LoG response (f3)
@pytest.mark.parametrize("nms,schedule", [("paper", None), ("26", None), ("paper", "band"), ("26", "band")])
def test_log_response_full_parity(c1_img, nms, schedule):
    """response="log" (reading R23): t_i^2 lap L(t_i) on the tensor cores (k_tc2: 2n
    sub-levels whose column products share one accumulator) and on the CUDA-core pair
    kernels (schedule="band") against the oracle's LoG stack: responses within 1e-4 of the
    peak, argmax, candidates, pruned blobs, counts and score under Eq. 2's parity rules."""
    tau = 0.1   # C1's tau / dt: LoG responses are ~1/dt times Eq. 2's
    s = _full_parity(c1_img, C1, nms=nms, tau=tau, response="log", schedule=schedule)
    assert s["n_oracle"] > 100
    det = mhfd.Detector(256, 256, threshold=tau, response="log", schedule=schedule, **C1)
    assert det.schedule("u8") == ("k_tc2" if schedule is None else "k_rows_pair+k_cols_pair<log>")


@pytest.mark.parametrize("bright", [False, True])
def test_log_response_k_tc2_multi_tile(bright):
    """LoG on k_tc2 over several 128-column x 224-row output tiles and NR-row row tiles
    (1024 x 512 u16, sigma 1-10, 10 scales, both polarities): LoG planes, v / argmax and
    the score against the oracle."""
    cfg = dict(min_sigma=1.0, max_sigma=10.0, num_scales=10)
    a = synth.em_tile_np(512, 1024, 1310, defocus=0.5, dose=300.0, bits=16)
    pol = "bright" if bright else "dark"
    det = mhfd.Detector(1024, 512, threshold=0.1, response="log", polarity=pol, **cfg)
    assert det.schedule("u16") == "k_tc2"
    t = torch.from_numpy(a.astype(np.int32)).cuda().to(torch.uint16)
    d = det.debug_dump(t, dog=True, cands=False)
    s = float(det.focus_score(t)[0])
    torch.cuda.synchronize()
    ref = oracle.detect(a, 1.0, 10.0, 10, 0.1, 0.5, dump=True, response="log", polarity=pol)
    eps = P.REL_EPS * float(ref["D"].max())
    assert float(np.abs(d["dog"][0].cpu().numpy() - ref["D"]).max()) <= eps
    assert float(np.abs(d["v"][0].cpu().numpy() - ref["v"]).max()) <= eps
    tie = P.scale_tie(ref["D"], eps)
    assert np.array_equal(d["idx"][0].cpu().numpy()[~tie], ref["idx"][~tie])
    P.assert_score(s, ref["count"])


def test_log_response_u16_ragged_and_degenerate():
    """LoG on u16, a ragged last row band (H = 200 with 256-row column tiles), a batch of
    two with a constant (degenerate) image: parity of v / argmax with the oracle for the
    real image, zeros and no blobs for the constant one."""
    cfg = dict(min_sigma=1.0, max_sigma=6.0, num_scales=5)
    a = synth.em_tile_np(200, 512, 1300, dose=300.0, bits=16)
    imgs = np.stack([a, np.full_like(a, 4321)])
    det = mhfd.Detector(512, 200, threshold=0.1, response="log", **cfg)
    t = torch.from_numpy(imgs.astype(np.int32)).to(torch.int32).cuda().to(torch.uint16)
    d = det.debug_dump(t, dog=True, cands=False)
    blobs, cnt, _ = det.detect(t)
    torch.cuda.synchronize()
    ref = oracle.detect(a, 1.0, 6.0, 5, 0.1, 0.5, dump=True, response="log")
    Pk = float(ref["D"].max())
    eps = P.REL_EPS * Pk
    assert float(np.abs(d["dog"][0].cpu().numpy() - ref["D"]).max()) <= eps
    assert float(np.abs(d["v"][0].cpu().numpy() - ref["v"]).max()) <= eps
    tie = P.scale_tie(ref["D"], eps)
    assert np.array_equal(d["idx"][0].cpu().numpy()[~tie], ref["idx"][~tie])
    assert float(d["dog"][1].abs().max()) == 0.0 and float(d["v"][1].abs().max()) == 0.0 and int(cnt[1]) == 0
    P.assert_score(int(cnt[0]), ref["count"])


@pytest.mark.parametrize("response", ["dog", "log"])
def test_two_pass_batch_chunks(response):
    """The two-pass schedules hold Rx for at most 8 images and run larger batches in
    chunks: a batch of 11 u16 tiles (different content, one constant) gives, image by
    image, the same kept blobs as 11 single-image calls."""
    imgs = [synth.em_tile_np(256, 512, 1400 + k, defocus=0.4 * (k % 5), dose=300.0, bits=16) for k in range(10)]
    imgs.append(np.full((256, 512), 900, np.uint16))
    batch = torch.from_numpy(np.stack(imgs).astype(np.int32)).cuda().to(torch.uint16)
    det = mhfd.Detector(512, 256, 1.0, 6.0, 5, threshold=0.1 if response == "log" else 0.1,
                        response=response)
    assert det.schedule("u16") == "k_tc2"
    blobs, cnt, _ = det.detect(batch)
    torch.cuda.synchronize()
    assert int(cnt[10]) == 0
    for k in range(11):
        b1, c1, _ = det.detect(batch[k:k + 1])
        torch.cuda.synchronize()
        n = int(c1[0])
        assert n == int(cnt[k]) and torch.equal(b1[0, :n], blobs[k, :n]), k


# ---------------------------------------------------------------- f32 input (f3)
@pytest.mark.parametrize("size,cfg", [(256, C1), (1000, C3)])
def test_f32_input_full_parity(size, cfg):
    """float32 images (reading R24): radix-select percentiles on real values (negative and
    positive, exact float32 bit patterns vs the oracle's sort), the stretch, and the rest of
    the path on the CUDA-core schedules (pair kernels at W = 256, k_scale_space at 1000)."""
    a = synth.em_tile_np(size, size, 1006, defocus=0.5, dose=300.0, bits=16).astype(np.float32)
    img = (a * np.float32(0.37) - np.float32(7000.25)).astype(np.float32)   # real values, both signs
    s = _full_parity(img, cfg)
    assert s["n_oracle"] > 50
    det = mhfd.Detector(size, size, threshold=_tau(cfg), **cfg)
    assert det.schedule("f32") == ("k_tc2" if size == 256 else "k_scale_space")


def test_f32_integer_valued_equals_u16():
    """Integer-valued float32 input gives the u16 result: the same percentiles (as values),
    the same stretch, hence the same blobs — a batch of two, one constant (degenerate)."""
    a = synth.em_tile_np(512, 512, 1007, dose=300.0, bits=16)
    imgs = np.stack([a, np.full_like(a, 1234)])
    det = mhfd.Detector(512, 512, threshold=_tau(C3), **C3)
    tu = torch.from_numpy(imgs.astype(np.int32)).cuda().to(torch.uint16)
    tf = torch.from_numpy(imgs.astype(np.float32)).cuda()
    bu, cu, _ = det.detect(tu)
    bf, cf, _ = det.detect(tf)
    torch.cuda.synchronize()
    assert int(cf[1]) == 0 and int(cu[1]) == 0
    n = int(cu[0])
    assert int(cf[0]) == n and torch.equal(bf[0, :n], bu[0, :n])


# ---------------------------------------------------------------- reflect boundary (f3)
@pytest.mark.parametrize("nms,response,schedule", [("paper", "dog", None), ("26", "dog", None),
                                                   ("paper", "dog", "band"), ("26", "dog", "band"),
                                                   ("paper", "log", None)])
def test_reflect_boundary_full_parity(c1_img, nms, response, schedule):
    """boundary="reflect" (reading R25): mirrored windows at all four edges, against the
    oracle's reflect blur; on k_tc (u8: mirrored rows by the window copies, mirrored
    columns inside the staged window) and on the two-pass kernels (schedule="band"; row
    staging pixel by pixel at the left/right edges, mirrored rows top/bottom); DoG in both
    NMS modes and the LoG response (two-pass)."""
    tau = 0.1 if response == "log" else None
    s = _full_parity(c1_img, C1, nms=nms, tau=tau, response=response, boundary="reflect", schedule=schedule)
    assert s["n_oracle"] > 100
    det = mhfd.Detector(256, 256, threshold=0.08, boundary="reflect", response=response, schedule=schedule, **C1)
    want = ("k_tc" if response == "dog" else "k_tc2") if schedule is None else "k_rows_pair+k_cols_pair"
    assert det.schedule("u8") == want


@pytest.mark.parametrize("kind,nms,response", [("u16", "paper", "dog"), ("u16", "26", "dog"), ("f32", "paper", "dog"),
                                               ("u16", "paper", "log")])
def test_reflect_k_tc2_full_parity(kind, nms, response):
    """Reflect on k_tc2 (u16 / f32 images, the LoG response): the stretched image is staged
    with mirrored margins (pg column groups, pr rows) so neither pass wraps; full parity on
    a 256 x 512 tile against the oracle's reflect blur."""
    a = synth.em_tile_np(256, 512, 1040, defocus=0.5, dose=300.0, bits=16)
    img = a if kind == "u16" else (a.astype(np.float32) * np.float32(0.25) + np.float32(3.5))
    tau = 0.1 if response == "log" else None
    det = mhfd.Detector(512, 256, threshold=0.1 if response == "log" else _tau(C1), boundary="reflect",
                        response=response, nms=nms, **C1)
    assert det.schedule(kind) == "k_tc2"
    s = _full_parity(img, C1, nms=nms, tau=tau, response=response, boundary="reflect")
    assert s["n_oracle"] > 100


def test_reflect_k_tc2_multi_tile():
    """Reflect on k_tc2 over many row and column tiles (1024 x 768 u16, sigma 1-10): full
    parity."""
    a = synth.em_tile_np(768, 1024, 1041, defocus=0.5, dose=300.0, bits=16)
    det = mhfd.Detector(1024, 768, threshold=_tau(C3), boundary="reflect", **C3)
    assert det.schedule("u16") == "k_tc2"
    s = _full_parity(a, C3, boundary="reflect")
    assert s["n_oracle"] > 1000


@pytest.mark.parametrize("w,h", [(1024, 1024), (2048, 1024)])
def test_reflect_k_tc_multi_tile(w, h):
    """Reflect on k_tc over many tiles: 1024^2 runs the level-split small-call variant
    (64 tiles, two level parts), 2048 x 1024 the whole-level variant; full parity."""
    img = synth.em_tile_np(h, w, 1030, defocus=0.5, dose=300.0, bits=8)
    det = mhfd.Detector(w, h, threshold=_tau(C3), boundary="reflect", **C3)
    assert det.schedule("u8") == "k_tc"
    s = _full_parity(img, C3, boundary="reflect")
    assert s["n_oracle"] > 1000


def test_reflect_differs_from_periodic_only_near_edges():
    """v under the two boundaries on the same pair kernels (u16): bit-identical farther
    than R_max from every edge (same staged values, same sums), different near the edges
    of a non-periodic image."""
    a16 = synth.em_tile_np(256, 512, 1008, dose=300.0, bits=16)
    img = torch.from_numpy(a16.astype(np.int32)).cuda().to(torch.uint16)
    res = []
    for bd in ("periodic", "reflect"):
        det = mhfd.Detector(512, 256, threshold=0.08, boundary=bd, schedule="band", **C1)   # both on the pair kernels
        assert det.schedule("u16") == "k_rows_pair+k_cols_pair"
        res.append(det.debug_dump(img, dog=False, cands=False)["v"][0].cpu())
    R = 25   # ceil(5 * 5)
    a, b = res
    assert torch.equal(a[R:-R, R:-R], b[R:-R, R:-R])
    assert float((a - b).abs().max()) > 1e-4


# ---------------------------------------------------------------- host-buffer path (e2e API)
@pytest.mark.parametrize("kind", ["u8", "u16", "f32", "u8-log"])
def test_focus_score_host_equals_device(kind):
    """mhfd_focus_score_host (pinned host batch, chunked H2D copies on a second stream
    overlapped with compute, ramped chunk sizes) returns exactly the device path's scores
    and counts: batch 11 with chunk 4 (chunks of 1, 2, 4, 4)."""
    B, n = 11, 512
    a = np.stack([synth.em_tile_np(n, n, 1500 + k, defocus=0.3 * (k % 4), dose=300.0,
                                   bits=8 if kind.startswith("u8") else 16) for k in range(B)])
    if kind == "u16":
        host = torch.from_numpy(a.astype(np.int32)).to(torch.uint16)
    elif kind == "f32":
        host = torch.from_numpy((a.astype(np.float32) * np.float32(0.5)) - np.float32(3.25))
    else:
        host = torch.from_numpy(a)
    host = host.pin_memory()
    det = mhfd.Detector(n, n, threshold=0.1 if kind == "u8-log" else _tau(C3),
                        response="log" if kind == "u8-log" else "dog", **C3)
    dev_scores, dev_counts = det.focus_score(host.cuda(), counts=True)
    hs, hc = det.focus_score_host(host, chunk=4, counts=True)
    torch.cuda.synchronize()
    assert torch.equal(hs, dev_scores.cpu()) and torch.equal(hc, dev_counts.cpu())
    assert float(hs.min()) > 0


def test_focus_score_host_pipelined_calls():
    """Back-to-back mhfd_focus_score_host calls without a synchronisation in between (the
    second call's copies overlap the first call's last chunks through the three staging
    slots, and it uses whole chunks): every call's scores equal the device path's, for
    two different batches and a ragged batch size."""
    n = 512
    mk = lambda seed, B: np.stack([synth.em_tile_np(n, n, seed + k, defocus=0.4 * (k % 5), dose=300.0, bits=8)
                                   for k in range(B)])
    batches = [torch.from_numpy(mk(1600, 13)).pin_memory(), torch.from_numpy(mk(1700, 9)).pin_memory()]
    det = mhfd.Detector(n, n, threshold=_tau(C3), **C3)
    ref = [det.focus_score(b.cuda()).cpu() for b in batches]
    torch.cuda.synchronize()
    order = [0, 1, 0, 1, 1, 0]
    outs = [(torch.empty(13, dtype=torch.float64).pin_memory(), torch.empty(13, dtype=torch.int32).pin_memory())
            for _ in order]
    for i, o in zip(order, outs):   # no synchronisation between the calls
        det.focus_score_host(batches[i], chunk=3, out=o)
    torch.cuda.synchronize()
    for i, (hs, hc) in zip(order, outs):
        B = batches[i].shape[0]
        assert torch.equal(hs[:B], ref[i]) and torch.equal(hc[:B].to(torch.float64), ref[i])


def test_downsample_pitched_buffers():
    """mhfd_downsample through the C ABI with row pitches wider than the rows (input and
    output), u8 factor 2 (vector path off: odd width) and u16 factor 3: bit-exact, and the
    padding bytes of the output rows are left untouched."""
    from paper_2108_12050_b200 import _abi
    lib = _abi.load()
    rng = np.random.default_rng(78)
    for dt, npd, code, bpp, f in ((torch.uint8, np.uint8, _abi.MHFD_U8, 1, 2), (torch.int16, np.uint16, _abi.MHFD_U16, 2, 3)):
        H, W, B = 37, 45, 2
        a = rng.integers(0, 256 if bpp == 1 else 65536, size=(B, H, W)).astype(npd)
        ip, OW, OH = (W * bpp + 32 + 15) // 16 * 16, -(-W // f), -(-H // f)
        op = (OW * bpp + 16 + 15) // 16 * 16
        src = torch.zeros((B, H, ip), dtype=torch.uint8)
        src.view(B, H, ip)[:, :, :W * bpp] = torch.from_numpy(a.view(np.uint8).reshape(B, H, W * bpp))
        src = src.cuda()
        dst = torch.full((B, OH, op), 0xAB, dtype=torch.uint8, device="cuda")
        st = lib.mhfd_downsample(src.data_ptr(), code, W, H, ip, f, dst.data_ptr(), op, B,
                                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert st == 0
        d = dst.cpu().numpy()
        for b in range(B):
            got = d[b, :, :OW * bpp].copy().view(npd).reshape(OH, OW)
            assert np.array_equal(got, oracle.downsample(a[b], f))
        assert (d[:, :, OW * bpp:] == 0xAB).all()


# ---------------------------------------------------------------- k_tc2 (two-pass tensor cores)
@pytest.mark.parametrize("bits,cfg,size", [(16, C3, 1024), (8, dict(min_sigma=1.0, max_sigma=20.0, num_scales=12), 1024),
                                           (16, C1, 512)])
def test_tc2_full_parity(bits, cfg, size):
    """k_tc2 (u16, and u8 with R_max 100 > k_tc's tile) in full against the oracle; and the
    CUDA-core pair kernels (schedule="band") on the same image agree with it within the
    parity tolerance."""
    img = synth.em_tile_np(size, size, 1011, defocus=0.5, dose=300.0, bits=bits)
    det = mhfd.Detector(size, size, threshold=_tau(cfg), **cfg)
    assert det.schedule(f"u{bits}") == "k_tc2"
    s = _full_parity(img, cfg)
    assert s["n_oracle"] > 500
    alt = mhfd.Detector(size, size, threshold=_tau(cfg), schedule="band", **cfg)
    t = _to_t(img) if bits == 8 else torch.from_numpy(img.astype(np.int32)).cuda().to(torch.uint16)
    va = det.debug_dump(t, dog=False, cands=False)["v"]
    vb = alt.debug_dump(t, dog=False, cands=False)["v"]
    torch.cuda.synchronize()
    assert float((va - vb).abs().max()) <= 2 * P.REL_EPS * float(vb.abs().max())


def test_tc2_batch_ragged_rows_and_degenerate():
    """k_tc2 with H not a multiple of its row tiles (NR) or of 256, a batch of 11 (> 8:
    chunked Rx), a constant image inside: image by image equal to single-image calls, the
    constant one all zero."""
    imgs = [synth.em_tile_np(400, 512, 1600 + k, defocus=0.3 * (k % 4), dose=300.0, bits=16) for k in range(10)]
    imgs.insert(4, np.full((400, 512), 1234, np.uint16))
    batch = torch.from_numpy(np.stack(imgs).astype(np.int32)).cuda().to(torch.uint16)
    det = mhfd.Detector(512, 400, 1.0, 6.0, 5, threshold=0.1)
    assert det.schedule("u16") == "k_tc2"
    blobs, cnt, _ = det.detect(batch)
    d = det.debug_dump(batch, dog=True, cands=False)
    torch.cuda.synchronize()
    assert int(cnt[4]) == 0 and float(d["v"][4].abs().max()) == 0.0 and float(d["dog"][4].abs().max()) == 0.0
    for k in range(11):
        b1, c1, _ = det.detect(batch[k:k + 1])
        torch.cuda.synchronize()
        n = int(c1[0])
        assert n == int(cnt[k]) and torch.equal(b1[0, :n], blobs[k, :n]), k
    ref = oracle.detect(imgs[7], 1.0, 6.0, 5, 0.1, 0.5, dump=True)
    eps = P.REL_EPS * float(ref["D"].max())
    assert float(np.abs(d["dog"][7].cpu().numpy() - ref["D"]).max()) <= eps
    P.assert_score(int(cnt[7]), ref["count"])


@pytest.mark.parametrize("size,G,bits", [(1024, 2, 8), (1024, 3, 8), (4096, 8, 8), (1024, 3, 16)])
def test_sharded_pruning_certificate(size, G, bits):
    """f2 sharded pruning (mhfd_prune_band; SURVEY §8(f) f2 "border-blob exchange"), the
    G ranks run one after another on this GPU.  (1) Synchronous rounds decide exactly
    like the default rounds: the whole image as one band (no truncated edge, certificate
    trivially 1) gives detect()'s count.  (2) Every certified band's count equals the
    number of the whole image's kept blobs in its rows, with the default halo and with a
    halo of one interaction radius D (which certifies fewer bands: the certificate must
    never claim a wrong count).  (3) With the default halo every band certifies on these
    EM tiles and the band counts sum to the image's count; the band candidate counts sum
    to the image's candidate count."""
    from paper_2108_12050_b200.dist import band_rows, halo_rows
    if bits == 8:
        img = synth.em_tile(size, size, 1004, defocus=0.5, dose=300.0, device="cuda")
        det = mhfd.Detector(size, size, threshold=0.09, **C3)
    else:   # u16 on k_tc2 at sigma 1-20 (R_max 100): the large-radius band path
        a = synth.em_tile_np(size, size, 1009, defocus=0.5, dose=300.0, bits=16)
        img = torch.from_numpy(a.astype(np.int32)).cuda().to(torch.uint16)
        det = mhfd.Detector(size, size, 1.0, 20.0, 12, threshold=0.1 * 19.0 / 12)
        assert det.schedule("u16") == "k_tc2"
    blobs, cnt, _ = det.detect(img)
    torch.cuda.synchronize()
    k_full = int(cnt[0])
    ys = blobs[0, :k_full, 1].cpu()
    c, n = det.detect_band(img, 0, size)
    kept, cert, nb = det.prune_band(c, int(n), 0, size, 0, size)
    assert int(kept[0]) == k_full and int(cert[0]) == 1 and int(nb[0]) == int(n)
    D = det.interaction_radius()
    assert D > 0
    for halo, expect_all in ((halo_rows(det), True), (D, False)):
        tot_kept, tot_n, ncert = 0, 0, 0
        for r in range(G):
            y0, y1 = band_rows(size, G, r)
            e0, e1 = max(0, y0 - halo), min(size, y1 + halo)
            c, n = det.detect_band(img, e0, e1)
            kept, cert, nb = det.prune_band(c, int(n), e0, e1, y0, y1)
            torch.cuda.synchronize()
            truth = int(((ys >= y0) & (ys < y1)).sum())
            if int(cert[0]):
                assert int(kept[0]) == truth, (halo, r, int(kept[0]), truth)
                ncert += 1
            tot_kept += int(kept[0])
            tot_n += int(nb[0])
        if expect_all:
            assert ncert == G and tot_kept == k_full
        full = det.debug_dump(img, dog=False, cands=True)
        assert tot_n == int(full["ncand"][0])


def test_focus_score_cuda_graph_capture():
    """The whole mhfd_focus_score call is stream-ordered with no host synchronisation, so
    it captures in a CUDA graph; replays give the eager result, also after the input is
    overwritten in place (the graph reads the buffer, not a snapshot)."""
    imgs = [synth.em_tile(1024, 1024, 1000 + g, defocus=1.0 * g, dose=300.0, device="cuda") for g in range(2)]
    det = mhfd.Detector(1024, 1024, threshold=0.09, overlap=0.5, **C3)
    ref = [float(det.focus_score(im[None])[0]) for im in imgs]
    buf = imgs[0][None].clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        det.focus_score(buf)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = det.focus_score(buf)
    for k in (0, 1, 0):
        buf.copy_(imgs[k][None])
        g.replay()
        torch.cuda.synchronize()
        assert float(out[0]) == ref[k], (k, float(out[0]), ref[k])
