"""World-size-2 gloo tests of the multi-GPU protocols (CPU): class sharding with the
feature all-gather and raw-output all-gather, and image-DP result gathering.  The
oracle stands in for the CUDA engine, so the collective flow and the merge order are
checked against a single-process run of the same oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_11441_b200.distributed import ClassShardPlan, detect_class_sharded, gather_detections, shard_images


class OracleEngine:
    def __init__(self):
        from oracle import dart_oracle as O

        self.O = O
        self.cfg = O.OracleConfig()
        self.P = O.build_params(self.cfg)
        self.num_queries = self.cfg.num_queries

    def prefix(self, images):
        img = images[0].numpy()
        flag = int(img.min() < 0 or img.max() > 1)  # like the device range flag: compute anyway, raise later
        l0, _, _ = self.O.backbone(self.P, self.cfg, np.clip(img, 0.0, 1.0))
        return torch.from_numpy(self.O.encoder_prefix(self.P, self.cfg, l0))[None], torch.tensor([flag], dtype=torch.int32)

    def decode(self, e1, names):
        texts = [self.O.text_embedding(self.P, self.cfg, n) for n in names]
        outs = [self.O.encdec(self.P, self.cfg, None, texts, e1=e1[w].numpy()) for w in range(e1.shape[0])]
        boxes = torch.from_numpy(np.stack([o[1] for o in outs]))
        scores = torch.from_numpy(np.stack([o[3] for o in outs]))
        pres = torch.from_numpy(np.stack([o[2] for o in outs]))
        return boxes, scores, pres

    def postprocess(self, boxes, scores, presence, names, cfg):
        return self.O.postprocess(boxes.numpy(), scores.numpy(), presence.numpy(), presence_thr=cfg["p"],
                                  score_thr=cfg["s"], cross_class=cfg["x"])

    @staticmethod
    def check_flags(flags):
        if flags:
            raise ValueError("image values must lie in [0, 1]")


NAMES = ["car", "person", "dog", "cat", "bus"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dart_oracle as O

        eng = OracleEngine()
        img, _ = O.scene(100 + rank, 64, num_classes=3)
        res = {}
        for xc in (False, True):
            cfg = {"p": 0.0, "s": 0.0, "x": xc}
            res[xc] = detect_class_sharded(eng, torch.from_numpy(img)[None], NAMES, cfg)
        mine = {i: f"img{i}@{rank}" for i in shard_images(5, rank, world)}
        merged = gather_detections(mine)
        q.put((rank, res, merged))
    finally:
        dist.destroy_process_group()


def test_class_sharded_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (res, merged)) for r, res, merged in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import dart_oracle as O

    eng = OracleEngine()
    for rank in range(world):
        img, _ = O.scene(100 + rank, 64, num_classes=3)
        for xc in (False, True):
            ref = O.run_detect(eng.P, eng.cfg, img, NAMES, presence_thr=0.0, score_thr=0.0, cross_class=xc)
            out = got[rank][0][xc]
            assert [(c, q) for c, q, *_ in out] == [(c, q) for c, q, *_ in ref]
            for a, b in zip(out, ref):
                np.testing.assert_allclose(a[2], b[2], rtol=1e-12)
                assert abs(a[3] - b[3]) < 1e-12
    assert got[0][1] == {0: "img0@0", 1: "img1@1", 2: "img2@0", 3: "img3@1", 4: "img4@0"}
    assert got[1][1] is None


def _bad_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dart_oracle as O

        eng = OracleEngine()
        img, _ = O.scene(100 + rank, 64, num_classes=3)
        if rank == 1:
            img = img.copy()
            img[0, 0, 0] = 1.5  # out of range on rank 1 only
        try:
            detect_class_sharded(eng, torch.from_numpy(img)[None], NAMES, {"p": 0.0, "s": 0.0, "x": False})
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_class_sharded_bad_image_raises_on_every_rank():
    """Reference model.py:432-433: a value outside [0, 1] raises ValueError.  In class-sharded
    mode the flag is reduced across ranks, so every rank raises (none is left in a collective)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: "image values must lie in [0, 1]", 1: "image values must lie in [0, 1]"}


def test_shard_plan_covers_all_classes():
    for n in (1, 3, 4, 80, 81):
        for w in (1, 2, 3, 8):
            plan = ClassShardPlan(n, w)
            covered = []
            for r in range(w):
                s, e = plan.bounds(r)
                assert 0 <= e - s <= plan.width
                covered.extend(range(s, e))
            assert covered == list(range(n))


def test_native_unpack_owner_arithmetic_matches_plan():
    """The owner / shard-start arithmetic of nccl_shard.cu:unpack_raw_kernel, restated, agrees
    with ClassShardPlan.bounds for every class of every (N, W) up to 9 ranks."""
    from paper_2603_11441_b200.distributed import ClassShardPlan

    for world in range(1, 10):
        for n in range(1, 90):
            plan = ClassShardPlan(n, world)
            base, extra = divmod(n, world)
            big = extra * (base + 1)
            for cls in range(n):
                owner = cls // (base + 1) if cls < big else extra + (cls - big) // (base if base > 0 else 1)
                start = owner * base + min(owner, extra)
                s, e = plan.bounds(owner)
                assert s == start and s <= cls < e and cls - start < plan.width


class _FakeEvent:
    def __init__(self, done_after):
        self.n, self.done_after = 0, done_after

    def query(self):
        self.n += 1
        return self.n > self.done_after


class _FakeLib:
    """dart_nccl_comm_check / _abort stand-ins: the communicator fails after `fail_after` checks."""

    def __init__(self, fail_after=None):
        self.checks, self.aborted, self.fail_after = 0, False, fail_after

    def dart_nccl_comm_check(self, ptr):
        self.checks += 1
        return 2 if self.aborted or (self.fail_after is not None and self.checks > self.fail_after) else 0

    def dart_nccl_comm_abort(self, ptr):
        self.aborted = True
        return 0

    def dart_last_error(self):
        return b"NCCL asynchronous error: remote process exited"


def _comm(lib):
    from paper_2603_11441_b200.distributed import NcclComm

    c = NcclComm.__new__(NcclComm)
    c.lib, c.ptr, c.world, c.rank = lib, 1, 2, 0
    return c


def test_nccl_wait_completes_aborts_on_error_and_times_out(monkeypatch):
    """NcclComm.wait (SURVEY section 5 failure detection): returns once the round's event completes
    while the communicator stays healthy; an asynchronous NCCL error or the timeout aborts the
    communicator (releasing ranks blocked in collectives) and raises RuntimeError."""
    from paper_2603_11441_b200 import _native

    monkeypatch.setattr(_native, "load", lambda: _FakeLib())
    ok = _FakeLib()
    _comm(ok).wait(_FakeEvent(3), timeout_s=10.0, poll_s=0.0)
    assert not ok.aborted and ok.checks >= 3
    bad = _FakeLib(fail_after=2)
    with pytest.raises(RuntimeError, match="failed"):
        _comm(bad).wait(_FakeEvent(10 ** 9), timeout_s=10.0, poll_s=0.0)
    assert bad.aborted
    slow = _FakeLib()
    with pytest.raises(RuntimeError, match="timed out"):
        _comm(slow).wait(_FakeEvent(10 ** 9), timeout_s=0.05, poll_s=0.001)
    assert slow.aborted
