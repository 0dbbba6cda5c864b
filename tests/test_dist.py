"""Multi-process host logic of the image-sharded path, world_size 2 over gloo (CPU).

Each rank scores its contiguous shard of a batch with the oracle (standing in for the
per-GPU kernels, which need a B200), gathers (count, score) with the same
`paper_2108_12050_b200.dist.gather_results` the bench uses over NCCL, and checks that
the gathered vector equals the single-process result (GPU-count invariance,
SPEC.md:339 analog) and that the shards partition the batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_12050_b200.dist import gather_results, shard


def test_shard_partitions():
    for n in (0, 1, 7, 64, 513):
        for w in (1, 2, 3, 8):
            parts = [shard(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, imgs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    s, e = shard(len(imgs), world, rank)
    counts = torch.tensor([oracle.detect(im, 1.0, 5.0, 5, 0.08, 0.5)["count"] for im in imgs[s:e]], dtype=torch.int32)
    scores = counts.to(torch.float64)
    g = gather_results(counts, scores)
    if rank == 0:
        q.put(g.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_world2_matches_single_process():
    import oracle
    import synth
    imgs = [synth.em_tile_np(64, 64, 1000 + b, dose=300.0) for b in range(4)]
    ref = np.array([oracle.detect(im, 1.0, 5.0, 5, 0.08, 0.5)["count"] for im in imgs], np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, imgs, q)) for r in range(2)]
    for p in procs:
        p.start()
    g = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert g.shape == (2, 2, 2)
    np.testing.assert_array_equal(g.reshape(-1, 2)[:, 0], ref)
    np.testing.assert_array_equal(g.reshape(-1, 2)[:, 1], ref)


# ---------------------------------------------------------------- single-image sharding (f2)
def _band_worker(rank, world, port, img, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2108_12050_b200.dist import band_rows, gather_candidates
    # the per-band candidates the GPU computes (mhfd_detect_band), here from the oracle:
    # the whole image's Eq. 3 candidates restricted to this rank's rows
    H = img.shape[0]
    ref = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5, dump=True)
    allc = oracle.nms_paper(ref["D"], 0.08)
    y0, y1 = band_rows(H, world, rank)
    mine = allc[(allc["y"] >= y0) & (allc["y"] < y1)]
    rec = torch.from_numpy(np.stack([mine["x"], mine["y"], mine["scale"]], 1).astype(np.int32))
    got, total = gather_candidates(rec, len(mine))
    if rank == 0:
        q.put((got.numpy(), total))
    dist.barrier()
    dist.destroy_process_group()


def test_band_sharding_world2_reassembles_raster_list():
    """Bands partition the rows; the all-gathered band lists are the whole image's
    candidate list in raster order, and pruning it gives the single-process result."""
    import oracle
    import synth
    from paper_2108_12050_b200.dist import band_rows
    for H in (64, 67):
        parts = [band_rows(H, 3, r) for r in range(3)]
        assert parts[0][0] == 0 and parts[-1][1] == H and all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    img = synth.em_tile_np(96, 80, 1003, dose=300.0)
    ref = oracle.detect(img, 1.0, 5.0, 5, 0.08, 0.5, dump=True)
    allc = oracle.nms_paper(ref["D"], 0.08)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, 2, port, img, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert total == len(allc)
    np.testing.assert_array_equal(got[:, 0], allc["x"])
    np.testing.assert_array_equal(got[:, 1], allc["y"])
    np.testing.assert_array_equal(got[:, 2], allc["scale"])
    keep = oracle.prune(allc, 1.0, 5.0, 5, 0.5)
    assert int(keep.sum()) == ref["count"]


def _overflow_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2108_12050_b200.dist import gather_candidates
    # rank 0 found 7 candidates but stored only 5 (its band list overflowed), rank 1
    # found 3 and stores them in a larger buffer: no hang, exact total, the records are
    # the first ones of the raster list
    n = 7 if rank == 0 else 3
    cap = 5 if rank == 0 else 9
    rec = torch.full((cap, 4), -1, dtype=torch.int32)
    for k in range(min(n, cap)):
        rec[k] = torch.tensor([k, 10 * rank, 0, 0], dtype=torch.int32)
    got, total = gather_candidates(rec, n)
    q.put((rank, got.numpy(), total))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_candidates_overflow_world2():
    """a band list truncated to its capacity must not desynchronise the
    all-gathers (each rank learns every rank's stored count), and the total stays exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overflow_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, got, total in res:
        assert total == 10
        assert got.shape == (8, 4)
        assert got[:5, 0].tolist() == [0, 1, 2, 3, 4] and (got[:5, 1] == 0).all()
        assert got[5:, 0].tolist() == [0, 1, 2] and (got[5:, 1] == 10).all()


# ---------------------------------------------------------------- sharded pruning (f2)
class _FakeDet:
    """Stands in for the Detector (the kernels need a B200): a fixed candidate set; a
    candidate is 'kept' iff its x is even, so band counts and the full-list count agree
    exactly as mhfd_prune_band's certified counts and mhfd_prune_candidates' do."""

    def __init__(self, H, cap, fail_rank=-1):
        rng = np.random.default_rng(5)
        ys = np.sort(rng.integers(0, H, 60))
        xs = rng.integers(0, 50, 60)
        self.rec = torch.tensor(np.stack([xs, ys, np.zeros(60), np.zeros(60)], 1), dtype=torch.int32)
        self.height, self.max_candidates, self.fail_rank = H, cap, fail_rank
        self.calls = []

    def interaction_radius(self):
        return 3

    def detect_band(self, image, y0, y1):
        m = self.rec[(self.rec[:, 1] >= y0) & (self.rec[:, 1] < y1)]
        cap = max(self.max_candidates, 1)
        out = torch.zeros((cap, 4), dtype=torch.int32)
        out[:min(len(m), cap)] = m[:cap]
        self.calls.append(("detect_band", y0, y1))
        return out, torch.tensor([len(m)], dtype=torch.int32)

    def prune_band(self, cands, n, e0, e1, y0, y1):
        c = cands[:n]
        inb = (c[:, 1] >= y0) & (c[:, 1] < y1)
        kept = int((inb & (c[:, 0] % 2 == 0)).sum())
        cert = 0 if dist.get_rank() == self.fail_rank else 1
        self.calls.append(("prune_band", e0, e1, y0, y1))
        return (torch.tensor([kept], dtype=torch.int32), torch.tensor([cert], dtype=torch.int32),
                torch.tensor([int(inb.sum())], dtype=torch.int32))

    def prune_candidates(self, allc, total):
        k = int((allc[:total, 0] % 2 == 0).sum())
        self.calls.append(("prune_candidates", total))
        return None, torch.tensor([k], dtype=torch.int32), torch.tensor([float(k)], dtype=torch.float64), \
            torch.tensor([0], dtype=torch.int32)


def _sharded_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2108_12050_b200.dist import focus_score_single_image_sharded
    det = _FakeDet(40, cap=100 if case != "overflow" else 30, fail_rank=1 if case == "fail" else -1)
    img = torch.zeros((40, 50), dtype=torch.uint8)
    cnt, score, sharded = focus_score_single_image_sharded(det, img)
    truth = int((det.rec[:, 0] % 2 == 0).sum()) if case != "overflow" else int((det.rec[:30, 0] % 2 == 0).sum())
    q.put((rank, cnt, score, sharded, truth, [c[0] for c in det.calls]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ok", "fail", "overflow"])
def test_sharded_pruning_world2(case):
    """dist.focus_score_single_image_sharded over gloo, world 2: certified bands -> the
    summed band counts (no candidate gather, no prune_candidates call); one failed
    certificate or more candidates than max_candidates (whose truncation needs the whole
    raster list) -> every rank falls back to the gather + replicated pruning, and all
    ranks return the same count."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, cnt, score, sharded, truth, calls in res:
        assert cnt == truth and score == float(truth)
        assert sharded == (case == "ok")
        assert ("prune_candidates" in calls) == (case != "ok")
