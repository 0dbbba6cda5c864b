"""Parity bookkeeping between the CUDA path and the oracle.

Tolerances are the north star's:
  * f32 responses within eps = 1e-4 * P of the oracle, P = the image's peak
    oracle response (max over pixels and planes of DoG);
  * blob sets and counts bit-exact, excluding the "ambiguous" set A of
    candidates within eps of the threshold or of a neighbour tie;
  * focus scores within 1e-3 relative.
"""
from __future__ import annotations

import math

import numpy as np

REL_EPS = 1e-4
SCORE_RTOL = 1e-3


def neighbour_max_2d(v: np.ndarray) -> np.ndarray:
    """max over the in-image 8-neighbourhood (-inf padding), centre excluded."""
    H, W = v.shape
    p = np.full((H + 2, W + 2), -np.inf)
    p[1:-1, 1:-1] = v
    m = np.full((H, W), -np.inf)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            if dy or dx:
                m = np.maximum(m, p[1 + dy:1 + dy + H, 1 + dx:1 + dx + W])
    return m


def neighbour_max_3d(D: np.ndarray) -> np.ndarray:
    n, H, W = D.shape
    p = np.full((n + 2, H + 2, W + 2), -np.inf)
    p[1:-1, 1:-1, 1:-1] = D
    m = np.full(D.shape, -np.inf)
    for di in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if di or dy or dx:
                    m = np.maximum(m, p[1 + di:1 + di + n, 1 + dy:1 + dy + H, 1 + dx:1 + dx + W])
    return m


def ambiguous_paper(v: np.ndarray, tau: float, eps: float) -> np.ndarray:
    """Pixels whose Eq. 3 candidacy f32 rounding could flip (bool H x W)."""
    m = neighbour_max_2d(v)
    relaxed = (v >= m - eps) & (v > tau - eps)
    return relaxed & ((np.abs(v - tau) <= eps) | (np.abs(v - m) <= eps))


def ambiguous_26(D: np.ndarray, tau: float, eps: float) -> np.ndarray:
    m = neighbour_max_3d(D)
    relaxed = (D >= m - eps) & (D > tau - eps)
    return relaxed & ((np.abs(D - tau) <= eps) | (np.abs(D - m) <= eps))


def scale_tie(D: np.ndarray, eps: float) -> np.ndarray:
    """Pixels whose top two scale responses are within eps (argmax may differ)."""
    if D.shape[0] < 2:
        return np.zeros(D.shape[1:], bool)
    s = np.sort(D, axis=0)
    return (s[-1] - s[-2]) <= eps


def blob_set(rows, with_scale=True):
    return {(int(r[0]), int(r[1]), int(r[2])) if with_scale else (int(r[0]), int(r[1])) for r in rows}


def gpu_rows(blobs, count):
    """(x, y, scale, response) from a (cap, 4) int32 tensor block."""
    b = blobs[:count].cpu().numpy()
    resp = b[:, 3].copy().view(np.float32)
    return [(int(x), int(y), int(s), float(r)) for (x, y, s), r in zip(b[:, :3], resp)]


def oracle_rows(bl):
    return [(int(b["x"]), int(b["y"]), int(b["scale"]), float(b["response"])) for b in bl]


def compare_candidates(gpu, ora, amb_xy: set, tie_xy: set, eps: float, mode: str):
    """Candidate sets equal outside A; scales equal unless tied; responses within eps.
    Returns a summary dict."""
    key = (lambda r: (r[0], r[1])) if mode == "paper" else (lambda r: (r[0], r[1], r[2]))
    g = {key(r): r for r in gpu}
    o = {key(r): r for r in ora}
    amb = (lambda k: (k[0], k[1]) in amb_xy) if mode == "paper" else (lambda k: k in amb_xy)
    g_out = {k for k in g if not amb(k)}
    o_out = {k for k in o if not amb(k)}
    diff = g_out ^ o_out
    assert not diff, f"{len(diff)} candidate mismatches outside the ambiguity band, e.g. {sorted(diff)[:5]}"
    for k in g_out:
        rg, ro = g[k], o[k]
        if mode == "paper" and (k[0], k[1]) not in tie_xy:
            assert rg[2] == ro[2], f"scale mismatch at {k}: gpu {rg[2]} oracle {ro[2]}"
        assert abs(rg[3] - ro[3]) <= eps, f"response at {k}: gpu {rg[3]} oracle {ro[3]} eps {eps}"
    flips = len((set(g) ^ set(o)))
    return {"n_gpu": len(g), "n_oracle": len(o), "ambiguous": len(amb_xy), "flips_in_band": flips}


def pruning_seeds(amb_xy, tie_xy, gpu_c, ora_c) -> list:
    """Seeds of A' for the kept-set comparison: the ambiguous candidates (rule 2) plus the
    candidates whose scale is exempt from comparison (top two scale responses within eps,
    rule 2's last clause).  Such a candidate's scale, hence its radius sqrt(2) t, may
    legitimately differ between the two sides, which changes its own kept record and the
    greedy decisions of the blobs it overlaps exactly as an ambiguous candidate does
    (reading R26)."""
    pts = {(int(k[0]), int(k[1])) for k in amb_xy}
    cand_xy = {(int(r[0]), int(r[1])) for r in list(gpu_c) + list(ora_c)}
    pts |= {(int(x), int(y)) for (x, y) in tie_xy if (int(x), int(y)) in cand_xy}
    return sorted(pts)


def compare_pruned(gpu, ora, amb_pts, rad_max: float, rad, mode: str):
    """Kept sets equal outside A' = A + {blobs within r_p + r_max of a member of A}
    (SURVEY.md §8(c) parity rule 4: an ambiguous candidate can only change the greedy
    decision of a blob it overlaps, i.e. one closer than r_p + r_a <= r_p + r_max).
    Nearest-member distances come from a k-d tree (full-size images have ~10^5 blobs)."""
    if not amb_pts:
        assert blob_set(gpu) == blob_set(ora), "pruned sets differ with no ambiguous candidate"
        return {"excluded": 0}
    from scipy.spatial import cKDTree
    tree = cKDTree(np.array([(p[0], p[1]) for p in amb_pts], np.float64))
    rad = np.asarray(rad, np.float64)

    def outside(rows):
        if not rows:
            return set()
        a = np.array([(r[0], r[1], r[2]) for r in rows], np.int64)
        d, _ = tree.query(a[:, :2].astype(np.float64), k=1)
        far = d > rad[a[:, 2]] + rad_max
        return {(int(x), int(y), int(s)) for (x, y, s) in a[far]}
    gk, ok = outside(gpu), outside(ora)
    diff = gk ^ ok
    assert not diff, f"{len(diff)} pruned-set mismatches outside A', e.g. {sorted(diff)[:5]}"
    excluded = len(gpu) + len(ora) - len(gk) - len(ok)
    return {"excluded": excluded}


def assert_prune_exact(gpu_cands, gpu_kept, cfg, overlap: float):
    """The pruning step in isolation, exactly: the oracle's greedy rule (f64 geometry on
    integer coordinates, grid early-out with identical decisions) applied to the CUDA
    path's own candidate list keeps exactly the blobs the CUDA path kept."""
    import oracle
    if not gpu_cands:
        assert not gpu_kept
        return 0
    rec = np.array([(r[0], r[1], r[2], 0) for r in gpu_cands], np.int32)
    keep = oracle.prune(oracle.blobs_from_records(rec), cfg["min_sigma"], cfg["max_sigma"], cfg["num_scales"],
                        overlap, grid=True)
    ref = {(int(x), int(y), int(s)) for (x, y, s, _), k in zip(rec, keep) if k}
    got = blob_set(gpu_kept)
    assert got == ref, f"pruning differs on the GPU's own candidates: {len(got ^ ref)} blobs"
    return len(ref)


def assert_score(s_gpu: float, s_oracle: float):
    assert abs(s_gpu - s_oracle) <= SCORE_RTOL * max(s_oracle, 1.0), (s_gpu, s_oracle)


def radii(min_t, max_t, n):
    t = [min_t + i * (max_t - min_t) / n for i in range(n + 1)]
    return [math.sqrt(2) * t[s] for s in range(n)]
