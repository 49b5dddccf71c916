"""Multi-GPU partitioning of the detection path, one process per GPU.

Two modes, both over `torch.distributed` (NCCL over NVLink on the B200 box; gloo in
the CPU tests, with an oracle-backed engine standing in for the CUDA one):

* image data parallelism -- images never interact: image i runs entirely on rank
  i mod W; no collective on the data path (`shard_images`, `gather_detections`).
* class sharding for large N -- after the class-agnostic backbone, classes are
  independent (reference model.py:559-564).  Each rank runs the backbone for its own
  image, the W level-0 feature blocks are all-gathered ([T, F0] per image), every rank
  decodes ITS class shard for all W images in one class-batched pass, and the raw
  outputs are all-gathered so each image's owner post-processes all N classes
  (identical semantics to run_batched, including cross-class NMS).

The engine is anything with `backbone(images) -> l0 [B,T,F0]`, `decode(l0, names) ->
(boxes [B,n,Q,4], scores [B,n,Q], presence [B,n])` and `postprocess(boxes, scores,
presence, names, cfg) -> list[Detection]` on torch tensors (see `NativeEngine`).
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


def detect_class_sharded(engine, image, class_names, cfg, group=None):
    """Class-sharded detection of one image per rank (W images in flight).

    `image` is this rank's [1, S, S, 3] tensor; returns the detections for it.  Data
    movement per round: all_gather of W x [T, F0] fp32 features, all_gather of the raw
    outputs W x [W, N/W, Q, 5] fp64 (both tiny next to the decode FLOPs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = ClassShardPlan(len(class_names), world)
    l0 = engine.backbone(image).contiguous()  # [1, T, F0]
    gathered = [torch.empty_like(l0) for _ in range(world)]
    dist.all_gather(gathered, l0, group=group)
    l0_all = torch.cat(gathered)  # [W, T, F0], image w owned by rank w
    s, e = plan.bounds(rank)
    width = plan.width
    Q = engine.num_queries
    boxes = torch.zeros((world, width, Q, 4), dtype=torch.float64, device=l0.device)
    scores = torch.zeros((world, width, Q), dtype=torch.float64, device=l0.device)
    pres = torch.zeros((world, width), dtype=torch.float64, device=l0.device)
    if e > s:
        b, sc, p = engine.decode(l0_all, class_names[s:e])
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
    return engine.postprocess(my_boxes, my_scores, my_pres, class_names, cfg)


class NativeEngine:
    """The CUDA engine for the sharded modes: one model handle on this rank's GPU."""

    def __init__(self, model, device=None):
        from .model import _device, native_handle

        self.model = model
        self.device = device or _device()
        self.handle = native_handle(model, self.device)
        self.num_queries = model.config.num_queries

    def backbone(self, images):
        from .model import backbone_forward_batch

        (l0, _, _), _ = backbone_forward_batch(self.model, images, check=True)
        return l0

    def decode(self, l0, names):
        import torch

        from .model import device_text, encdec_forward_device, text_encode

        emb = text_encode(self.model, list(names))
        text = device_text(self.model, emb.stack(list(names)), self.device)
        B = int(l0.shape[0])
        raw = encdec_forward_device(self.model, l0, text, B, len(names), with_query_features=False)
        n, Q = len(names), self.num_queries
        return (raw.d_boxes.reshape(B, n, Q, 4), raw.d_score_logits.reshape(B, n, Q),
                raw.d_presence_logits.reshape(B, n))

    def postprocess(self, boxes, scores, presence, names, cfg):
        from .pipeline import detections_from_result, postprocess_device

        res = postprocess_device(boxes, scores, presence, cfg, self.model)
        return detections_from_result(res.to_host(), boxes.cpu().numpy(), list(names), cfg.cross_class_nms)
