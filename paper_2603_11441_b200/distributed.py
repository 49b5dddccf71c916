"""Multi-GPU partitioning of the detection path, one process per GPU.

Two modes, both over `torch.distributed` (NCCL over NVLink on the B200 box; gloo in
the CPU tests, with an oracle-backed engine standing in for the CUDA one):

* image data parallelism -- images never interact: image i runs entirely on rank
  i mod W; no collective on the data path (`shard_images`, `gather_detections`).
* class sharding for large N -- after the class-agnostic backbone and the class-independent
  enc-dec prefix (input projection + encoder layer-0 self-attention, model.py:513-517),
  classes are independent (model.py:559-564).  Each rank runs backbone + prefix for its own
  image, the W prefix outputs e1 ([T, d] per image) are all-gathered, every rank decodes
  ITS class shard for all W images in one class-batched pass, and the raw outputs are
  all-gathered so each image's owner post-processes all N classes (identical semantics to
  run_batched, including cross-class NMS).

The engine is anything with `prefix(images) -> (e1 [B,T,d], flags int32 [1])`,
`decode(e1, names) -> (boxes [B,n,Q,4], scores [B,n,Q], presence [B,n])`,
`postprocess(boxes, scores, presence, names, cfg) -> list[Detection]` and
`check_flags(int)` on torch tensors (see `NativeEngine`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ClassShardPlan:
    """Contiguous, balanced class ranges: rank r decodes names[start(r):stop(r)]."""

    n_classes: int
    world: int

    def bounds(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.n_classes, self.world)
        start = rank * base + min(rank, extra)
        return start, start + base + (1 if rank < extra else 0)

    @property
    def width(self) -> int:
        """Padded shard width used for the all-gather of raw outputs."""
        return -(-self.n_classes // self.world)


def image_owner(index: int, world: int) -> int:
    return index % world


def shard_images(n_images: int, rank: int, world: int) -> list[int]:
    """Image-DP: the image indices rank `rank` processes."""
    return [i for i in range(n_images) if image_owner(i, world) == rank]


def gather_detections(local: dict, group=None) -> dict | None:
    """Image-DP result merge: {image index: detections} from every rank to rank 0."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, local, group=group)
    if dist.get_rank(group) != 0:
        return None
    merged = {}
    for part in out:
        merged.update(part)
    return dict(sorted(merged.items()))


def class_sharded_raw(engine, image, class_names, group=None):
    """The collective part of `detect_class_sharded`, fully asynchronous on the device:
    returns this rank's image's raw outputs over ALL classes (boxes [N, Q, 4], score logits
    [N, Q], presence logits [N], float64) and the rank-reduced status flags (int32 [1])."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = ClassShardPlan(len(class_names), world)
    e1, flags = engine.prefix(image)  # [1, T, d], int32 [1] (device, asynchronous)
    e1 = e1.contiguous()
    gathered = [torch.empty_like(e1) for _ in range(world)]
    dist.all_gather(gathered, e1, group=group)
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    e1_all = torch.cat(gathered)  # [W, T, d], image w owned by rank w
    s, e = plan.bounds(rank)
    width = plan.width
    Q = engine.num_queries
    boxes = torch.zeros((world, width, Q, 4), dtype=torch.float64, device=e1.device)
    scores = torch.zeros((world, width, Q), dtype=torch.float64, device=e1.device)
    pres = torch.zeros((world, width), dtype=torch.float64, device=e1.device)
    if e > s:
        b, sc, p = engine.decode(e1_all, class_names[s:e])
        boxes[:, : e - s] = b
        scores[:, : e - s] = sc
        pres[:, : e - s] = p
    packed = torch.cat([boxes.reshape(world, width, Q * 4), scores, pres[..., None]], dim=2)  # [W, width, 5Q+1]
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    rows = []
    for r in range(world):
        rs, re_ = plan.bounds(r)
        rows.append(parts[r][rank, : re_ - rs])  # classes rs..re_ of MY image, from rank r
    mine = torch.cat(rows)  # [N, 5Q+1]
    n = len(class_names)
    my_boxes = mine[:, : 4 * Q].reshape(n, Q, 4).contiguous()
    my_scores = mine[:, 4 * Q: 5 * Q].contiguous()
    my_pres = mine[:, 5 * Q].contiguous()
    return my_boxes, my_scores, my_pres, flags


def detect_class_sharded(engine, image, class_names, cfg, group=None):
    """Class-sharded detection of one image per rank (W images in flight).

    `image` is this rank's [1, S, S, 3] tensor; returns the detections for it.  Each rank
    runs the backbone and the class-independent enc-dec prefix (model.py:513-517) of its own
    image; the W prefix outputs e1 [T, d] fp32 are all-gathered (5.3 MB per image at full
    size; fp32 so the sharded outputs stay bitwise equal to run_batched); every rank decodes
    ITS class shard for all W images in one class-batched pass; the raw outputs
    (W x [W, N/W, Q, 5] fp64) are all-gathered so each image's owner post-processes all N
    classes.  The backbone status flags are MAX-reduced across ranks with the features and
    checked only after the results reach the host, so a bad image raises on every rank (no
    rank left blocked in a collective) and there is no extra host synchronisation."""
    my_boxes, my_scores, my_pres, flags = class_sharded_raw(engine, image, class_names, group)
    dets = engine.postprocess(my_boxes, my_scores, my_pres, class_names, cfg)  # host results (synchronises)
    engine.check_flags(int(flags.reshape(-1)[0].item()))
    return dets


class NativeEngine:
    """The CUDA engine for the sharded modes: one model handle on this rank's GPU.  Every
    method but `postprocess` only enqueues work on the current stream (no host sync)."""

    def __init__(self, model, device=None):
        from .model import _device, native_handle

        self.model = model
        self.device = device or _device()
        self.handle = native_handle(model, self.device)
        self.lib = self.handle.lib
        self.num_queries = model.config.num_queries
        self._bufs = {}

    def _buffers(self, B: int):
        import torch

        b = self._bufs.get(B)
        if b is None:
            cfg, dev = self.model.config, self.device
            T, g = cfg.tokens, cfg.grid
            b = self._bufs[B] = {
                "l0": torch.empty((B, T, cfg.fpn_dims[0]), device=dev, dtype=torch.float32),
                "l1": torch.empty((B, (g // 2) ** 2, cfg.fpn_dims[1]), device=dev, dtype=torch.float32),
                "l2": torch.empty((B, (g // 4) ** 2, cfg.fpn_dims[2]), device=dev, dtype=torch.float32),
            }
        return b

    def prefix(self, images):
        """images [B, S, S, 3] device float32 -> (e1 [B, T, d] fp32, flags int32 [1]): the
        backbone and the class-independent enc-dec prefix (dart_backbone + dart_encdec_prefix)."""
        import torch

        from . import _native
        from .model import _stream_ptr

        cfg = self.model.config
        imgs = images.to(device=self.device, dtype=torch.float32).contiguous()
        B = int(imgs.shape[0])
        b = self._buffers(B)
        flags = torch.zeros((1,), device=self.device, dtype=torch.int32)
        e1 = torch.empty((B, cfg.tokens, cfg.text_dim), device=self.device, dtype=torch.float32)
        st = _stream_ptr(self.device)
        with torch.cuda.device(self.device):
            _native.check(self.lib.dart_backbone(self.handle.ptr, imgs.data_ptr(), B, b["l0"].data_ptr(),
                                                 b["l1"].data_ptr(), b["l2"].data_ptr(), flags.data_ptr(), st))
            _native.check(self.lib.dart_encdec_prefix(self.handle.ptr, None, B, e1.data_ptr(), st))
        return e1, flags

    def decode(self, e1, names, out=None):
        """e1 [B, T, d] fp32 (device) x names -> raw outputs (boxes [B,n,Q,4], score logits [B,n,Q],
        presence logits [B,n]) float64 on the device (dart_encdec_from_prefix)."""
        import torch

        from . import _native
        from .model import _stream_ptr, device_text, text_encode

        emb = text_encode(self.model, list(names))
        text = device_text(self.model, emb.stack(list(names)), self.device)
        B, n, Q = int(e1.shape[0]), len(names), self.num_queries
        if out is None:
            out = (torch.empty((B, n, Q, 4), device=self.device, dtype=torch.float64),
                   torch.empty((B, n, Q), device=self.device, dtype=torch.float64),
                   torch.empty((B, n), device=self.device, dtype=torch.float64))
        boxes, scores, pres = out
        with torch.cuda.device(self.device):
            _native.check(self.lib.dart_encdec_from_prefix(
                self.handle.ptr, e1.contiguous().data_ptr(), B, text.contiguous().data_ptr(), n, boxes.data_ptr(),
                scores.data_ptr(), pres.data_ptr(), None, _stream_ptr(self.device)))
        return boxes, scores, pres

    def postprocess_device(self, boxes, scores, presence, cfg):
        from .pipeline import postprocess_device

        return postprocess_device(boxes, scores, presence, cfg, self.model)

    def postprocess(self, boxes, scores, presence, names, cfg):
        from .pipeline import detections_from_result

        res = self.postprocess_device(boxes, scores, presence, cfg)
        return detections_from_result(res.to_host(), boxes.cpu().numpy(), list(names), cfg.cross_class_nms)

    @staticmethod
    def check_flags(flags: int) -> None:
        from .model import raise_for_flags

        raise_for_flags(flags)


class NcclComm:
    """A communicator of the C ABI's own NCCL helpers (dart_nccl_*, include/dart_b200.h): the
    class-sharded round without torch.distributed on the data path.  The 128-byte unique id is
    created on rank 0 and handed to the other ranks over `group` (any torch.distributed backend;
    host bytes only), or passed in directly (`unique_id`)."""

    def __init__(self, world: int, rank: int, group=None, unique_id: bytes | None = None, device=None):
        import ctypes

        import torch

        from . import _native

        self.lib = _native.load()
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if not self.lib.dart_nccl_available():
            raise RuntimeError("dart_nccl_*: libnccl.so.2 could not be opened")
        if unique_id is None:
            buf = (ctypes.c_uint8 * 128)()
            if rank == 0:
                _native.check(self.lib.dart_nccl_unique_id(buf))
            if world > 1:
                import torch.distributed as dist

                obj = [bytes(buf)]
                dist.broadcast_object_list(obj, src=0, group=group)
                buf = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        else:
            buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        out = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.dart_nccl_comm_create(buf, world, rank, ctypes.byref(out)))
        self.ptr = out.value
        self.world, self.rank = world, rank

    def check(self) -> None:
        """Raise if the communicator has an asynchronous error (dead peer, broken link); never blocks."""
        from . import _native

        _native.check(self.lib.dart_nccl_comm_check(self.ptr))

    def abort(self) -> None:
        """ncclCommAbort: release every collective this rank is blocked in; later calls fail."""
        if self.ptr:
            self.lib.dart_nccl_comm_abort(self.ptr)

    def wait(self, event, timeout_s: float = 60.0, poll_s: float = 1e-3) -> None:
        """Block until `event` (a torch.cuda.Event recorded after a round) completes, polling the
        communicator's asynchronous error; on an error or after `timeout_s` the communicator is
        aborted (so no rank stays blocked in a collective) and RuntimeError is raised."""
        import time

        deadline = time.monotonic() + timeout_s
        while not event.query():
            try:
                self.check()
            except Exception as e:
                self.abort()
                raise RuntimeError(f"class-sharded round failed: {e}") from e
            if time.monotonic() > deadline:
                self.abort()
                raise RuntimeError(f"class-sharded round timed out after {timeout_s:.1f} s (communicator aborted)")
            time.sleep(poll_s)
        self.check()

    def close(self):
        if self.ptr:
            self.lib.dart_nccl_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def class_sharded_raw_native(engine, comm: NcclComm, images, class_names, timeout_s: float | None = None):
    """`class_sharded_raw` through the C ABI (dart_class_sharded): one call per round, all
    collectives inside the library.  images [B, S, S, 3] (this rank's); returns boxes [B, N, Q, 4],
    score logits [B, N, Q], presence logits [B, N] (float64, device) of this rank's images over
    all N classes, and the rank-reduced flags (int32 [1]).  Asynchronous on the current stream,
    unless `timeout_s` is given: then the round is awaited with NcclComm.wait (asynchronous NCCL
    errors and the timeout abort the communicator and raise)."""
    import torch

    from . import _native
    from .model import _stream_ptr, device_text, text_encode

    names = list(class_names)
    imgs = images.to(device=engine.device, dtype=torch.float32).contiguous()
    B, N, Q = int(imgs.shape[0]), len(names), engine.num_queries
    text = device_text(engine.model, text_encode(engine.model, names).stack(names), engine.device).contiguous()
    boxes = torch.empty((B, N, Q, 4), device=engine.device, dtype=torch.float64)
    scores = torch.empty((B, N, Q), device=engine.device, dtype=torch.float64)
    pres = torch.empty((B, N), device=engine.device, dtype=torch.float64)
    flags = torch.zeros((1,), device=engine.device, dtype=torch.int32)
    with torch.cuda.device(engine.device):
        _native.check(engine.lib.dart_class_sharded(engine.handle.ptr, comm.ptr, imgs.data_ptr(), B, text.data_ptr(), N,
                                                    boxes.data_ptr(), scores.data_ptr(), pres.data_ptr(),
                                                    flags.data_ptr(), _stream_ptr(engine.device)))
        if timeout_s is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(engine.device))
            comm.wait(ev, timeout_s)
    return boxes, scores, pres, flags
