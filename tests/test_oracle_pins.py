"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these tests re-types the oracle's own formula or re-calls the routine
it uses.  Each pins one oracle function to something independent of it:
a value the paper/spec prints, a closed form, a textbook/library routine that
computes the same definition by other means (numpy FFT of the paper's own
Fourier-domain formula, scipy.ndimage, torch max_pool2d), brute force, or an
invariant.  Each test names the oracle step (DESIGN.md §4 pin table).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.ndimage as ndi
import torch

import oracle
import synth


# ---------------------------------------------------------------- percentiles
def test_percentiles_spec_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "percentile_spec_example.json")))
    img = np.arange(1000, dtype=np.uint16).reshape(25, 40)
    lo, hi = oracle.percentiles(img, g["sat_low"], g["sat_high"])
    assert (lo, hi) == (g["lo"], g["hi"])
    f = oracle.stretch(img, lo, hi)
    assert f.flat[g["pixel"]] == pytest.approx(g["stretched_num"] / g["stretched_den"], abs=1e-15)
    assert f.min() == 0.0 and f.max() == 1.0


@pytest.mark.parametrize("dtype,shape,seed", [(np.uint8, (37, 53), 1), (np.uint16, (64, 61), 2),
                                              (np.uint8, (256, 256), 3), (np.uint16, (1, 1), 4)])
def test_percentiles_vs_counting_definition(dtype, shape, seed):
    # lo = min{v : #(p <= v) > k}, hi = min{v : #(p <= v) > N-1-k}: the rank
    # definition evaluated by counting (no sort), compared with the oracle's sort.
    rng = np.random.default_rng(seed)
    top = 255 if dtype == np.uint8 else 65535
    img = rng.integers(0, top + 1, size=shape).astype(dtype)
    img.flat[: max(1, img.size // 50)] = top  # a saturated tail
    N = img.size
    for f_lo, f_hi in [(0.00175, 0.00175), (0.0, 0.0), (0.01, 0.05)]:
        k_lo, k_hi = int(math.floor(f_lo * N)), int(math.floor(f_hi * N))
        vals = np.unique(img)
        cum = np.array([(img <= v).sum() for v in vals])
        lo = int(vals[np.argmax(cum > k_lo)])
        hi = int(vals[np.argmax(cum > N - 1 - k_hi)])
        assert oracle.percentiles(img, f_lo, f_hi) == (lo, hi)


def test_stretch_affine_invariance_and_monotone():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 200, size=(40, 50)).astype(np.uint16)
    lo, hi = oracle.percentiles(img)
    f = oracle.stretch(img, lo, hi)
    img2 = (img.astype(np.int64) * 7 + 1234).astype(np.uint16)
    lo2, hi2 = oracle.percentiles(img2)
    f2 = oracle.stretch(img2, lo2, hi2)
    np.testing.assert_allclose(f2, f, atol=1e-15)
    order = np.argsort(img.ravel(), kind="stable")
    assert np.all(np.diff(f.ravel()[order]) >= 0)


def test_stretch_degenerate_is_zero():
    img = synth.constant_image(9, 11, 77)
    lo, hi = oracle.percentiles(img)
    assert lo == hi == 77
    assert np.all(oracle.stretch(img, lo, hi) == 0.0)


# ---------------------------------------------------------------- Gaussian
def test_gaussian_center_value(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "gaussian_center.json")))
    assert oracle.gaussian_2d(0.0, 0.0, g["sigma"]) == pytest.approx(g["value"], rel=1e-15)
    # integral of the continuous kernel is 1 (numerical quadrature, independent of the taps)
    xs = np.linspace(-12, 12, 2401)
    G = np.array([[oracle.gaussian_2d(x, y, 1.7) for x in xs[::8]] for y in xs[::8]])
    assert G.sum() * (xs[8] - xs[0]) ** 2 == pytest.approx(1.0, abs=1e-6)


@pytest.mark.parametrize("t", [0.8, 1.0, 1.9, 4.6, 10.0, 28.55])
def test_gaussian_taps_closed_form(t):
    w = oracle.gaussian_taps(t)
    R = (len(w) - 1) // 2
    assert R == math.ceil(6 * t)
    assert w.sum() == pytest.approx(1.0, abs=1e-14)
    np.testing.assert_array_equal(w, w[::-1])
    d = np.arange(-R, R + 1)
    # ratio to the centre tap is exp(-d^2 / 2t^2): sigma = t
    np.testing.assert_allclose(w / w[R], np.exp(-d * d / (2 * t * t)), rtol=1e-13)


# ---------------------------------------------------------------- blur
def _paper_fft_blur(f, t):
    """The paper's own formula L = F^-1{F{G}.F{I}} with the full-size
    periodic, *unrenormalised* continuous kernel G(x,y,t) of PAPER.md:136."""
    H, W = f.shape
    y = np.minimum(np.arange(H), H - np.arange(H)).astype(np.float64)
    x = np.minimum(np.arange(W), W - np.arange(W)).astype(np.float64)
    G = np.exp(-(y[:, None] ** 2 + x[None, :] ** 2) / (2 * t * t)) / (2 * np.pi * t * t)
    return np.real(np.fft.ifft2(np.fft.fft2(G) * np.fft.fft2(f)))


@pytest.mark.parametrize("shape,t", [((64, 64), 1.0), ((96, 80), 2.5), ((128, 128), 5.0), ((130, 70), 1.9)])
def test_blur_matches_paper_fft_formula(shape, t):
    rng = np.random.default_rng(11)
    f = rng.random(shape)
    L = oracle.blur(f, t)
    # differences: sampling renormalisation (1.1e-8 at t=1) + truncation at 6t (2e-9)
    np.testing.assert_allclose(L, _paper_fft_blur(f, t), atol=3e-8, rtol=0)


@pytest.mark.parametrize("t", [1.0, 2.8, 6.4])
def test_blur_matches_scipy_gaussian_filter(t):
    rng = np.random.default_rng(12)
    f = rng.random((160, 150))
    R = math.ceil(6 * t)
    ref = ndi.gaussian_filter(f, sigma=t, mode="wrap", radius=R)
    np.testing.assert_allclose(oracle.blur(f, t), ref, atol=1e-13, rtol=0)


@pytest.mark.parametrize("shape,t", [((16, 16), 1.0), ((17, 23), 1.3), ((17, 23), 2.0)])
def test_blur_matches_bruteforce_2d(shape, t):
    # non-separable 2-D periodic sum of the renormalised sampled G(x,y,t) of PAPER.md:136
    rng = np.random.default_rng(13)
    f = rng.random(shape)
    R = math.ceil(6 * t)
    K = np.array([[math.exp(-(a * a + b * b) / (2 * t * t)) for b in range(-R, R + 1)] for a in range(-R, R + 1)])
    K /= K.sum()
    ref = np.zeros_like(f)
    for a in range(-R, R + 1):
        for b in range(-R, R + 1):
            ref += K[a + R, b + R] * np.roll(f, shift=(-a, -b), axis=(0, 1))
    np.testing.assert_allclose(oracle.blur(f, t), ref, atol=1e-14, rtol=0)


def test_blur_impulse_and_constant():
    t, H, W = 2.0, 41, 45
    f = np.zeros((H, W)); f[0, 0] = 1.0
    L = oracle.blur(f, t)
    R = math.ceil(6 * t)
    # impulse response at offset (a, b) is proportional to G(a, b, t)
    for (a, b) in [(0, 0), (1, 0), (0, 3), (5, 7), (-4, 2)]:
        ratio = L[a % H, b % W] / L[0, 0]
        assert ratio == pytest.approx(oracle.gaussian_2d(a, b, t) / oracle.gaussian_2d(0, 0, t), rel=1e-12)
    assert L.sum() == pytest.approx(1.0, abs=1e-14)
    c = np.full((H, W), 0.37)
    np.testing.assert_allclose(oracle.blur(c, t), 0.37, atol=1e-15)


def test_blur_semigroup():
    # G(a) * G(b) = G(sqrt(a^2+b^2)) for the continuous kernel; the sampled one
    # agrees to ~1e-6 relative at sigma >= 1
    rng = np.random.default_rng(14)
    f = ndi.gaussian_filter(rng.random((128, 128)), 2.0, mode="wrap")
    a, b = 1.5, 2.0
    np.testing.assert_allclose(oracle.blur(oracle.blur(f, a), b), oracle.blur(f, math.hypot(a, b)),
                               atol=2e-6 * np.ptp(f))


# ---------------------------------------------------------------- DoG (Eq. 2)
@pytest.mark.parametrize("s", [2.0, 3.0, 5.0])
def test_dog_closed_form_gaussian_blob(s):
    # I = 1 - A exp(-r^2/2s^2)  =>  centre DoG_i = t_i A s^2 (1/(s^2+t_i^2) - 1/(s^2+t_{i+1}^2))
    H = W = 160
    A, n, tmin, tmax = 0.5, 10, 1.0, 10.0
    f = synth.gaussian_blob_float(H, W, 80, 80, s, A)
    D = oracle.dog_stack(f, tmin, tmax, n, rows=(80, 81))[:, 0, 80]
    t = np.linspace(tmin, tmax, n + 1)
    ref = t[:-1] * A * s * s * (1 / (s * s + t[:-1] ** 2) - 1 / (s * s + t[1:] ** 2))
    np.testing.assert_allclose(D, ref, atol=5e-6 * np.abs(ref).max(), rtol=0)
    assert int(np.argmax(D)) == int(np.argmax(ref))


@pytest.mark.parametrize("r", [3.0, 5.0, 8.0, 12.0])
def test_dog_closed_form_disk(r):
    # dark disk of radius r, depth 1: centre L(t) = exp(-r^2/2t^2), so
    # DoG_i = t_i (exp(-r^2/2t_{i+1}^2) - exp(-r^2/2t_i^2)); the area-sampled disk
    # agrees to a few % of the peak and has the same argmax
    H = W = 128
    n, tmin, tmax = 10, 1.0, 10.0
    f = synth.disks_float(H, W, [(64.5, 64.5, r)], contrast=1.0)   # centred on pixel (64, 64)
    D = oracle.dog_stack(f, tmin, tmax, n, rows=(64, 65))[:, 0, 64]
    t = np.linspace(tmin, tmax, n + 1)
    ref = t[:-1] * (np.exp(-r * r / (2 * t[1:] ** 2)) - np.exp(-r * r / (2 * t[:-1] ** 2)))
    assert int(np.argmax(D)) == int(np.argmax(ref))
    np.testing.assert_allclose(D, ref, atol=0.03 * ref.max())


def test_dog_linearity_and_constant():
    rng = np.random.default_rng(15)
    f = rng.random((64, 72))
    D1 = oracle.dog_stack(f, 1.0, 3.0, 3)
    np.testing.assert_allclose(oracle.dog_stack(2.5 * f, 1.0, 3.0, 3), 2.5 * D1, atol=1e-13)
    np.testing.assert_allclose(oracle.dog_stack(np.full((40, 40), 0.3), 1.0, 3.0, 3), 0.0, atol=1e-15)


def test_dog_at_matches_stack():
    rng = np.random.default_rng(16)
    f = rng.random((70, 66))
    D = oracle.dog_stack(f, 1.0, 4.0, 4)
    for (y, x) in [(0, 0), (69, 65), (35, 12), (3, 60)]:
        np.testing.assert_allclose(oracle.dog_at(f, 1.0, 4.0, 4, y, x), D[:, y, x], atol=1e-13)


def test_scale_grid():
    t = oracle.scale_grid(1.0, 10.0, 10)          # n+1 levels, t_{n+1} = max_t
    np.testing.assert_allclose(t, 1.0 + 0.9 * np.arange(11), atol=1e-15)
    assert oracle.scale_grid(1.0, 2.0, 1).tolist() == [1.0, 2.0]


# ---------------------------------------------------------------- NMS, Eq. 3
def test_scale_argmax_tie_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "argmax_tie.json")))
    D = np.array(g["responses"], np.float64).reshape(-1, 1, 1)
    v, idx = oracle.scale_argmax(D)
    assert v[0, 0] == g["value"] and idx[0, 0] + 1 == g["index_1based"]


def _paper_nms_via_maxpool(D, tau, strict):
    """Eq. 3 with the paper's own primitive: torch argmax over scales (first on
    ties) and comparison against maxpool_2d(3,3)."""
    Dt = torch.from_numpy(D)
    v, idx = Dt.max(dim=0)
    idx = torch.from_numpy(np.argmax(D, axis=0))
    mp = torch.nn.functional.max_pool2d(v[None, None], 3, 1, 1)[0, 0]
    cand = (v == mp) & (v > tau)
    if strict:
        # strictly greater than every neighbour: maxpool of the plane with the centre removed
        vp = torch.nn.functional.pad(v[None, None], (1, 1, 1, 1), value=-math.inf)[0, 0]
        H, W = v.shape
        nb = torch.stack([vp[1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
                          for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dy, dx) != (0, 0)]).max(0).values
        cand = (v > nb) & (v > tau)
    ys, xs = np.nonzero(cand.numpy())
    return [(int(x), int(y), int(idx[y, x]), float(v[y, x])) for y, x in zip(ys, xs)]


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("strict", [False, True])
def test_nms_paper_vs_maxpool(seed, strict):
    n = 1 + seed % 5
    D = synth.random_stack(n, 8, 8, seed, levels=4) if seed < 3 else np.random.default_rng(seed).random((n, 32, 29))
    tau = 0.5 if seed % 2 else -1.0
    got = [(int(b["x"]), int(b["y"]), int(b["scale"]), float(b["response"])) for b in oracle.nms_paper(D, tau, strict)]
    assert got == _paper_nms_via_maxpool(D, tau, strict)


def test_nms_paper_vs_scipy_maximum_filter():
    rng = np.random.default_rng(21)
    D = rng.random((5, 48, 40))
    v = D.max(0)
    mf = ndi.maximum_filter(v, size=3, mode="constant", cval=-np.inf)
    ys, xs = np.nonzero((v == mf) & (v > 0.3))
    got = oracle.nms_paper(D, 0.3)
    assert list(zip(got["y"], got["x"])) == list(zip(ys, xs))


def test_nms_bruteforce_small_cases():
    # single peak -> one hit; constant plane -> no strict maxima
    D = np.zeros((1, 5, 5)); D[0, 2, 2] = 1.0
    b = oracle.nms_paper(D, 0.0)
    assert [(int(b["x"][0]), int(b["y"][0]))] == [(2, 2)] and len(b) == 1
    C = np.full((3, 8, 8), 0.25)
    assert len(oracle.nms_paper(C, 0.0, strict=True)) == 0
    assert len(oracle.nms_paper(C, 0.0, strict=False)) == 64   # maxpool equality holds everywhere
    assert len(oracle.nms_paper(C, 0.25)) == 0                  # threshold is strict (v > tau)


def _nms26_scipy(D, tau, strict):
    fp = np.ones((3, 3, 3), bool); fp[1, 1, 1] = False
    mf = ndi.maximum_filter(D, footprint=fp, mode="constant", cval=-np.inf)
    c = (D > mf) if strict else (D >= mf)
    c &= D > tau
    i, y, x = np.nonzero(c)
    order = np.lexsort((i, x, y))
    return list(zip(x[order], y[order], i[order]))


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("strict", [False, True])
def test_nms26_vs_scipy(seed, strict):
    D = synth.random_stack(2 + seed, 8, 8, 100 + seed, levels=3) if seed < 3 else \
        np.random.default_rng(seed).random((4, 24, 21))
    got = oracle.nms_26(D, 0.5, strict)
    assert list(zip(got["x"], got["y"], got["scale"])) == _nms26_scipy(D, 0.5, strict)


# ---------------------------------------------------------------- pruning
def test_lens_closed_form(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "lens_unit.json")))
    assert oracle.lens_fraction(g["d"], g["r1"], g["r2"]) == pytest.approx(g["fraction"], rel=1e-14)
    assert oracle.lens_fraction(0.5, 3.0, 1.0) == 1.0     # containment
    assert oracle.lens_fraction(4.0, 3.0, 1.0) == 0.0     # tangent externally
    assert oracle.lens_fraction(9.0, 3.0, 1.0) == 0.0     # disjoint


@pytest.mark.parametrize("d,r1,r2", [(1.3, 1.0, 1.5), (4.2, 3.0, 2.0), (2.0, 2.5, 0.9), (10.0, 7.0, 6.5)])
def test_lens_vs_grid_integration(d, r1, r2):
    m = 1500
    xs = np.linspace(-r1, r1, m)
    X, Y = np.meshgrid(xs, xs)
    inside = (X ** 2 + Y ** 2 <= r1 * r1) & ((X - d) ** 2 + Y ** 2 <= r2 * r2)
    area = inside.sum() * (xs[1] - xs[0]) ** 2
    frac = area / (math.pi * min(r1, r2) ** 2)
    assert oracle.lens_fraction(d, r1, r2) == pytest.approx(frac, abs=4e-3)
    assert oracle.lens_fraction(d, r1, r2) == oracle.lens_fraction(d, r2, r1)


def _blobs(rows):
    b = np.zeros(len(rows), oracle.BLOB_DTYPE)
    for k, (x, y, s) in enumerate(rows):
        b[k]["x"], b[k]["y"], b[k]["scale"], b[k]["response"] = x, y, s, 1.0
    return b


def test_prune_chain_case():
    # t_A > t_B > t_C; A overlaps B, B overlaps C, A and C disjoint -> keep {A, C}
    t = oracle.scale_grid(1.0, 10.0, 10)     # radius sqrt(2) t
    A, B, C = (0, 0, 9), (11, 0, 6), (19, 0, 3)
    rA, rB, rC = (math.sqrt(2) * t[s] for s in (9, 6, 3))
    assert oracle.lens_fraction(11, rA, rB) > 0.5 and oracle.lens_fraction(8, rB, rC) > 0.5
    assert oracle.lens_fraction(19, rA, rC) == 0.0
    keep = oracle.prune(_blobs([C, A, B]), 1.0, 10.0, 10, 0.5)
    assert keep.tolist() == [True, True, False]


def test_prune_greedy_characterisation():
    # the greedy result is the unique set K with: no two kept blobs overlap by > o,
    # and every removed blob overlaps a higher-priority kept blob by > o
    rng = np.random.default_rng(31)
    rows = list({(int(rng.integers(0, 60)), int(rng.integers(0, 60)), int(rng.integers(0, 10))) for _ in range(150)})
    b = _blobs(rows)
    t = oracle.scale_grid(1.0, 10.0, 10)
    for o in (0.0, 0.1, 0.5, 0.9):
        keep = oracle.prune(b, 1.0, 10.0, 10, o)
        pri = sorted(range(len(rows)), key=lambda k: (-rows[k][2], rows[k][1], rows[k][0]))
        rank = {k: r for r, k in enumerate(pri)}

        def frac(i, j):
            d = math.hypot(rows[i][0] - rows[j][0], rows[i][1] - rows[j][1])
            return oracle.lens_fraction(d, math.sqrt(2) * t[rows[i][2]], math.sqrt(2) * t[rows[j][2]])
        K = [k for k in range(len(rows)) if keep[k]]
        for i in K:
            for j in K:
                if i < j:
                    assert frac(i, j) <= o
        for r in range(len(rows)):
            if not keep[r]:
                assert any(frac(r, k) > o and rank[k] < rank[r] for k in K)
    assert oracle.prune(b, 1.0, 10.0, 10, 1.0).all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_prune_grid_equals_bruteforce(seed):
    """oracle_prune_grid (exact distance early-out, cells >= 2 r_max) keeps exactly the
    blobs the O(n^2) oracle_prune keeps: clustered lists with negative-offset coordinates
    (cells anchored at the minimum), every overlap value, and the chain case."""
    rng = np.random.default_rng(100 + seed)
    centres = rng.integers(-40, 400, size=(30, 2))
    rows = set()
    for cx, cy in centres:   # dense clusters: many overlapping pairs, long suppression chains
        for _ in range(60):
            rows.add((int(cx + rng.normal(0, 9)), int(cy + rng.normal(0, 9)), int(rng.integers(0, 10))))
    rows = sorted(rows)
    b = _blobs(rows)
    for o in (0.0, 0.1, 0.5, 0.9, 1.0):
        brute = oracle.prune(b, 1.0, 10.0, 10, o)
        grid = oracle.prune(b, 1.0, 10.0, 10, o, grid=True)
        assert np.array_equal(brute, grid), o
        if o < 1.0:
            assert 0 < brute.sum() < len(rows)
    A, B, C = (0, 0, 9), (11, 0, 6), (19, 0, 3)
    assert oracle.prune(_blobs([C, A, B]), 1.0, 10.0, 10, 0.5, grid=True).tolist() == [True, True, False]
    assert oracle.prune(_blobs([]), 1.0, 10.0, 10, 0.5, grid=True).size == 0


def test_detect_grid_prune_equals_default():
    img = synth.em_tile_np(128, 160, 1010, dose=300.0)
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.3)
    g = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.3, grid_prune=True)
    assert a["count"] == g["count"] > 0 and np.array_equal(a["blobs"], g["blobs"])


# ---------------------------------------------------------------- end to end
def test_detect_constant_is_zero():
    r = oracle.detect(synth.constant_image(64, 64, 200), 1.0, 5.0, 5, 0.0, 0.5)
    assert r["count"] == 0 and r["n_candidates"] == 0


@pytest.mark.parametrize("r", [4.0, 6.0, 9.0])
def test_detect_isolated_disk(r):
    # one dark disk, noise-free: exactly one blob, at the centre, at sigma ~ r/sqrt(2)
    n, tmin, tmax = 10, 1.0, 10.0
    dt = (tmax - tmin) / n
    img = synth.disk_image(96, 96, 48.5, 48.5, r, contrast=0.6, bits=16)
    res = oracle.detect(img, tmin, tmax, n, 0.1 * dt, 0.5)
    assert res["count"] == 1
    b = res["blobs"][0]
    assert (int(b["x"]), int(b["y"])) == (48, 48)
    t_hat = tmin + int(b["scale"]) * dt
    assert abs(t_hat + dt / 2 - r / math.sqrt(2)) <= 0.61 + 1e-9   # SURVEY A.9; north_star "sigma ~ r/sqrt(2)"


def test_detect_separated_disks():
    centres = [(24.5 + 48 * i, 24.5 + 48 * j) for i in range(3) for j in range(3)]
    rad = [3.0, 4.0, 5.0, 6.0, 7.0, 5.5, 4.5, 3.5, 6.5]
    f = synth.disks_float(144, 144, [(cy, cx, r) for (cy, cx), r in zip(centres, rad)], contrast=0.6)
    img = synth.quantise(torch.from_numpy(f), 16).numpy().astype(np.uint16)
    res = oracle.detect(img, 1.0, 10.0, 10, 0.09, 0.5)
    got = sorted((int(b["y"]), int(b["x"])) for b in res["blobs"])
    assert got == sorted((int(cy), int(cx)) for cy, cx in centres)


@pytest.mark.parametrize("nms", ["paper", "26"])
def test_detect_defocus_monotone_noise_free(nms):
    # count falls with defocus; noise-free, every tau >= 0
    counts = []
    for s in [0.0, 1.0, 2.0, 3.0, 4.0]:
        img = synth.em_tile_np(192, 192, 1000, defocus=s, dose=None, bits=16)
        counts.append(oracle.detect(img, 1.0, 10.0, 10, 0.09, 0.5, nms=nms)["count"])
    assert all(a > b for a, b in zip(counts, counts[1:])), counts


def test_detect_affine_invariance():
    img = synth.em_tile_np(96, 112, 7, bits=8).astype(np.uint16)
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5)
    b = oracle.detect((img * 5 + 321).astype(np.uint16), 1.0, 5.0, 5, 0.08, 0.5)
    assert a["count"] == b["count"]
    np.testing.assert_array_equal(a["blobs"][["x", "y", "scale"]], b["blobs"][["x", "y", "scale"]])


def test_detect_transpose_equivariance():
    # the detector is isotropic: candidates of I^T are the transposed candidates of I
    img = synth.em_tile_np(80, 96, 8, bits=8)
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 1.0)
    b = oracle.detect(np.ascontiguousarray(img.T), 1.0, 5.0, 5, 0.08, 1.0)
    sa = sorted((int(p["x"]), int(p["y"]), int(p["scale"])) for p in a["blobs"])
    sb = sorted((int(p["y"]), int(p["x"]), int(p["scale"])) for p in b["blobs"])
    assert sa == sb and len(sa) > 10


def test_detect_shift_equivariance_interior():
    # periodic blur => a circular shift moves every interior candidate by the shift
    img = synth.em_tile_np(96, 96, 9, bits=8)
    dy, dx = 13, -21
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 1.0)
    b = oracle.detect(np.roll(img, (dy, dx), axis=(0, 1)), 1.0, 5.0, 5, 0.08, 1.0)

    def interior(bl, sy, sx):
        out = set()
        for p in bl:
            y, x = (int(p["y"]) + sy) % 96, (int(p["x"]) + sx) % 96
            if 2 <= y < 94 and 2 <= x < 94 and 2 <= int(p["y"]) < 94 and 2 <= int(p["x"]) < 94:
                out.add((y, x, int(p["scale"])))
        return out
    A = interior(a["blobs"], dy, dx)
    B = {(int(p["y"]), int(p["x"]), int(p["scale"])) for p in b["blobs"]}
    assert A and A <= B


# ---------------------------------------------------------------- polarity
def test_bright_polarity_equals_dark_on_inverted_image():
    """bright(I) == dark(M - I): the inverted image's nearest-rank percentiles are
    (M - hi, M - lo), its stretch is 1 - I', and the unit-sum blur maps 1 - I' to 1 - L,
    so its Eq. 2 stack is exactly the negated one (up to f64 rounding)."""
    for bits, M in ((8, 255), (16, 65535)):
        img = synth.em_tile_np(96, 112, 1000, dose=300.0, bits=bits)
        inv = (M - img.astype(np.int64)).astype(img.dtype)
        a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5, dump=True, polarity="bright")
        b = oracle.detect(inv, 1.0, 5.0, 5, 0.08, 0.5, dump=True, polarity="dark")
        assert (a["lo"], a["hi"]) == (M - b["hi"], M - b["lo"])
        peak = float(np.abs(a["D"]).max())
        assert float(np.abs(a["D"] - b["D"]).max()) <= 1e-12 * peak
        ka = {(int(r["x"]), int(r["y"]), int(r["scale"])) for r in a["blobs"]}
        kb = {(int(r["x"]), int(r["y"]), int(r["scale"])) for r in b["blobs"]}
        assert ka == kb and a["count"] == b["count"] > 10


def test_bright_polarity_negates_dark_response():
    """Polarity only flips the sign of Eq. 2: D_bright = -D_dark on the same image."""
    img = synth.em_tile_np(80, 80, 1001, dose=300.0, bits=8)
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5, dump=True, polarity="bright")
    b = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5, dump=True, polarity="dark")
    assert np.array_equal(a["D"], -b["D"])


@pytest.mark.parametrize("r", [4.0, 7.0])
def test_bright_disk_detected_only_with_bright_polarity(r):
    """A bright disk on a dark background: one blob at the centre with bright polarity,
    at the scale the dark-disk closed form gives (|t + dt/2 - r/sqrt 2| <= 0.61);
    with the paper's dark polarity its centre responds negatively and is not a blob."""
    n, tmin, tmax = 10, 1.0, 10.0
    dt = (tmax - tmin) / n
    dark = synth.disk_image(96, 96, 48.5, 48.5, r, contrast=0.6, bits=16)
    bright = (65535 - dark.astype(np.int64)).astype(np.uint16)
    res = oracle.detect(bright, tmin, tmax, n, 0.1 * dt, 0.5, polarity="bright")
    assert res["count"] == 1
    b = res["blobs"][0]
    assert (int(b["x"]), int(b["y"])) == (48, 48)
    assert abs(tmin + int(b["scale"]) * dt + dt / 2 - r / math.sqrt(2)) <= 0.61 + 1e-9
    res_dark = oracle.detect(bright, tmin, tmax, n, 0.1 * dt, 0.5, polarity="dark")
    assert (48, 48) not in {(int(q["x"]), int(q["y"])) for q in res_dark["blobs"]}


# ---------------------------------------------------------------- downsampling (f4)
# PAPER.md:401 ("downsampling, by bilinear interpolation"); reading R22.

def test_downsample_identity_and_constant():
    rng = np.random.default_rng(3)
    for dt in (np.uint8, np.uint16):
        a = rng.integers(0, np.iinfo(dt).max + 1, size=(13, 17), dtype=dt)
        assert np.array_equal(oracle.downsample(a, 1), a)                     # SPEC.md:52 factor 1
    c = np.full((4, 4), 128, np.uint8)
    assert np.array_equal(oracle.downsample(c, 2), np.full((2, 2), 128, np.uint8))


def test_downsample_ramp_hand_values():
    # 4x4 ramp, factor 2, evaluated by hand at the sample centres x = 2X + 1/2:
    # each output is the mean of one 2x2 block, e.g. (0 + 10 + 40 + 50) / 4 = 25
    a = (np.arange(16).reshape(4, 4) * 10).astype(np.uint8)
    assert oracle.downsample(a, 2).tolist() == [[25, 45], [105, 125]]
    # factor 3 on 4x4: ceil -> 2x2; samples at x = 1, 4 -> columns 1, 3 (clamped)
    assert oracle.downsample(a, 3).tolist() == [[50, 70], [130, 150]]
    # a half-way value rounds up: (1 + 2 + 1 + 2) / 4 = 1.5 -> 2
    assert oracle.downsample(np.array([[1, 2], [1, 2]], np.uint8), 2).tolist() == [[2]]


@pytest.mark.parametrize("f", [2, 3, 4, 5])
def test_downsample_matches_torch_bilinear(f):
    # library routine: torch bilinear, align_corners=False (half-pixel centres, edge clamp)
    # on divisible shapes, in f64, rounded half up
    rng = np.random.default_rng(10 + f)
    a = rng.integers(0, 65536, size=(6 * f, 7 * f), dtype=np.uint16)
    t = torch.nn.functional.interpolate(torch.from_numpy(a.astype(np.float64))[None, None], scale_factor=1.0 / f,
                                        mode="bilinear", align_corners=False, recompute_scale_factor=False)
    ref = np.floor(t[0, 0].numpy() + 0.5).astype(np.uint16)
    assert np.array_equal(oracle.downsample(a, f), ref)


@pytest.mark.parametrize("shape,f", [((13, 17), 2), ((13, 17), 3), ((9, 20), 4), ((31, 29), 5), ((8, 8), 8)])
def test_downsample_closed_form_integer_factor(shape, f):
    # for an integer factor the sample x = X f + (f - 1)/2 is a pixel (odd f) or the
    # midpoint of two (even f): output = that pixel, or the rounded-half-up mean of the
    # 2 x 2 block, indices clamped to the image (brute force over a ragged shape)
    rng = np.random.default_rng(sum(shape) + f)
    a = rng.integers(0, 256, size=shape, dtype=np.uint8)
    H, W = shape
    out = oracle.downsample(a, f)
    assert out.shape == (-(-H // f), -(-W // f))
    for Y in range(out.shape[0]):
        for X in range(out.shape[1]):
            if f % 2:
                y, x = min(Y * f + (f - 1) // 2, H - 1), min(X * f + (f - 1) // 2, W - 1)
                want = int(a[y, x])
            else:
                y0, x0 = min(Y * f + f // 2 - 1, H - 1), min(X * f + f // 2 - 1, W - 1)
                y1, x1 = min(y0 + 1, H - 1), min(x0 + 1, W - 1)
                s = int(a[y0, x0]) + int(a[y0, x1]) + int(a[y1, x0]) + int(a[y1, x1])
                want = (s + 2) // 4
            assert int(out[Y, X]) == want, (Y, X)


# ---------------------------------------------------------------- LoG response (f3)
# PAPER.md:156-163 (Eq. 1, "t^2 lap L"); reading R23.

def test_log_taps_moments():
    for t in (1.0, 1.9, 4.3, 10.0):
        w, w2 = oracle.log_taps(t)
        R = (len(w) - 1) // 2
        d = np.arange(-R, R + 1, dtype=np.float64)
        assert abs(w2.sum()) < 1e-15                        # zero sum: constants respond 0
        assert abs((w2 * d * d).sum() / 2 - 1.0) < 1e-5     # second-moment normalisation
        assert np.allclose(w2, w2[::-1], atol=0)            # symmetric
        assert w2[R] < 0 and w2[0] > 0                      # negative centre lobe, positive tails


def test_log_constant_image_is_zero():
    f = np.full((48, 40), 0.37)
    assert np.abs(oracle.log_stack(f, 1.0, 5.0, 5)).max() < 1e-14


@pytest.mark.parametrize("s", [2.0, 3.5, 5.0])
def test_log_gaussian_blob_closed_form(s):
    # dark Gaussian blob 1 - A exp(-r^2 / 2 s^2): the blurred image is
    # 1 - A s^2/(s^2+t^2) exp(-r^2 / 2(s^2+t^2)), so at the centre
    # t^2 lap L = 2 A t^2 s^2 / (s^2 + t^2)^2 (positive: dark blobs respond positively)
    A, N = 0.6, 160
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    r2 = (yy - N // 2) ** 2 + (xx - N // 2) ** 2
    f = 1.0 - A * np.exp(-r2 / (2 * s * s))
    mn, mx, n = 1.0, 10.0, 10
    D = oracle.log_stack(f, mn, mx, n, rows=(N // 2, N // 2 + 1))[:, 0, N // 2]
    t = oracle.scale_grid(mn, mx, n)[:n]
    want = 2 * A * t ** 2 * s ** 2 / (s * s + t ** 2) ** 2
    # sampled vs continuous: the discrete sums differ from the integrals by Poisson
    # aliasing, whose leading term decays like exp(-2 pi^2 t^2 s^2 / (t^2 + s^2)) (the
    # product of the two sampled Gaussians' spectra); 1e3 covers its polynomial prefactor
    # (measured 2.2e-5 of the peak at t = 1, s = 2); the support ceil(6t) cuts the
    # second-derivative taps' tails, t^2 x 2 int_{6t}^inf |g''| ~ 12 e^-18 / sqrt(2 pi)
    # = 7.4e-8 (measured <= 7.2e-8 of the peak): 2e-7
    alias = np.exp(-2 * np.pi ** 2 * t ** 2 * s ** 2 / (t ** 2 + s ** 2))
    assert np.all(np.abs(D - want) <= (2e-7 + 1e3 * alias) * want.max())
    assert int(np.argmax(D)) == int(np.argmax(want))       # scale selection: t ~ s


def test_log_separable_equals_2d_definition():
    # the 2-D operator sum_{a,b} (w2(a) w(b) + w(a) w2(b)) f(y+a, x+b), periodic,
    # evaluated directly at a few pixels of a random image
    rng = np.random.default_rng(8)
    f = rng.random((22, 26))
    mn, mx, n = 1.0, 2.0, 2
    D = oracle.log_stack(f, mn, mx, n)
    t = oracle.scale_grid(mn, mx, n)
    for i in range(n):
        w, w2 = oracle.log_taps(t[i])
        R = (len(w) - 1) // 2
        K = np.outer(w2, w) + np.outer(w, w2)      # K[a, b]: a along y, b along x
        for (y, x) in ((0, 0), (5, 17), (21, 25), (11, 3)):
            acc = 0.0
            for a in range(-R, R + 1):
                for b in range(-R, R + 1):
                    acc += K[a + R, b + R] * f[(y + a) % 22, (x + b) % 26]
            assert abs(D[i, y, x] - t[i] ** 2 * acc) < 1e-13


def test_log_detect_single_disk():
    # end to end with response="log": one dark disk -> exactly one blob at its centre,
    # at the scale where t^2 lap L of the disk peaks (t ~ r / sqrt 2 for a disk)
    N, r = 128, 8.0
    yy, xx = np.mgrid[0:N, 0:N].astype(np.float64)
    f = np.where((yy - 64) ** 2 + (xx - 64) ** 2 <= r * r, 60, 200).astype(np.uint8)
    res = oracle.detect(f, 1.0, 10.0, 10, 0.05, 0.5, response="log")
    assert res["count"] == 1
    b = res["blobs"][0]
    assert (int(b["x"]), int(b["y"])) == (64, 64)
    t = oracle.scale_grid(1.0, 10.0, 10)
    assert abs(t[int(b["scale"])] - r / np.sqrt(2)) <= 0.9 + 1e-9


# ---------------------------------------------------------------- f32 input (f3)
# SURVEY §8(f) f3 "f32 input dtype with a float-quantile select"; reading R24.

def test_f32_percentiles_nearest_rank_and_integer_agreement():
    rng = np.random.default_rng(21)
    a = rng.integers(0, 256, size=(40, 37), dtype=np.uint8)
    # integer-valued floats: the same ranks and the same stretch as the u8 image
    lo_i, hi_i = oracle.percentiles(a, 0.05, 0.05)
    lo_f, hi_f = oracle.percentiles(a.astype(np.float32), 0.05, 0.05)
    assert (lo_f, hi_f) == (float(lo_i), float(hi_i))
    assert np.array_equal(oracle.stretch(a.astype(np.float32), lo_f, hi_f), oracle.stretch(a, lo_i, hi_i))
    # real values: sort-based nearest rank written out, negatives included
    x = rng.normal(0.0, 3.0, size=(33, 29)).astype(np.float32)
    s = np.sort(x.ravel().astype(np.float64))
    k = int(np.floor(0.00175 * x.size))
    assert oracle.percentiles(x) == (s[k], s[x.size - 1 - k])
    # affine invariance of the stretch on real values: a*x + b, a > 0
    y = (2.0 * x.astype(np.float64) + 5.0).astype(np.float32)
    ly, hy = oracle.percentiles(y)
    lx, hx = oracle.percentiles(x)
    assert np.allclose(oracle.stretch(y, ly, hy), oracle.stretch(x, lx, hx), atol=1e-6)


def test_f32_detect_equals_u8_on_integer_floats():
    img = synth.em_tile_np(96, 96, 1000, dose=300.0, bits=8)
    a = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5)
    b = oracle.detect(img.astype(np.float32), 1.0, 5.0, 5, 0.08, 0.5)
    assert a["count"] == b["count"] and np.array_equal(a["blobs"], b["blobs"])
    assert np.frombuffer(np.uint32(b["lo"]).tobytes(), np.float32)[0] == float(a["lo"])


# ---------------------------------------------------------------- reflect boundary (f3)
# SURVEY §8(f) f3 "reflect boundary"; reading R25 (half-sample symmetric, scipy 'reflect').

@pytest.mark.parametrize("t", [1.0, 2.5, 4.0])
def test_reflect_blur_matches_scipy(t):
    rng = np.random.default_rng(31)
    f = rng.random((57, 61))
    R = oracle.radius(t)
    ref = ndi.gaussian_filter(f, t, mode="reflect", radius=R)
    assert np.abs(oracle.blur(f, t, boundary="reflect") - ref).max() < 1e-13


def _mirror_tile(f):
    # the half-sample-symmetric extension of f is the periodic extension of this 2H x 2W tile
    top = np.concatenate([f, f[:, ::-1]], 1)
    return np.concatenate([top, top[::-1, :]], 0)


@pytest.mark.parametrize("stack", ["dog", "log"])
def test_reflect_equals_periodic_on_mirror_tile(stack):
    # reflect-boundary responses of f = periodic responses of the mirrored 2H x 2W tile
    # restricted to f (a different formulation of the same boundary rule)
    rng = np.random.default_rng(32)
    f = rng.random((26, 30))
    fn = oracle.dog_stack if stack == "dog" else oracle.log_stack
    a = fn(f, 1.0, 2.0, 3, boundary="reflect")
    b = fn(_mirror_tile(f), 1.0, 2.0, 3)[:, :26, :30]
    assert np.abs(a - b).max() < 1e-13
    # constant images respond 0 under either boundary
    assert np.abs(fn(np.full((26, 30), 0.4), 1.0, 2.0, 3, boundary="reflect")).max() < 1e-14


def test_reflect_boundary_changes_only_the_edges():
    # far from the edges (> R_max) the two boundaries agree exactly
    rng = np.random.default_rng(33)
    f = rng.random((80, 84))
    a = oracle.dog_stack(f, 1.0, 3.0, 2, boundary="reflect")
    b = oracle.dog_stack(f, 1.0, 3.0, 2)
    R = oracle.radius(3.0)
    assert np.abs(a[:, R:-R, R:-R] - b[:, R:-R, R:-R]).max() < 1e-15
    assert np.abs(a - b).max() > 1e-6
