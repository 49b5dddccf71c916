"""Detector model API, B200 edition: a drop-in for the reference's `dart.model`
(/root/reference/pkg/src/dart/model.py) on the detection path.

Host-side (Python, NumPy): configuration, deterministic weight init, serialization,
the text-embedding cache and structural edits -- cheap bookkeeping the reference also
does on the host.  Device-side: `backbone_forward` and `encdec_forward` hand the
weights to libdart_b200.so once per (model, device) and run the sm_100a kernels
through the C ABI (include/dart_b200.h).  There is no CPU compute path.
"""

from __future__ import annotations

import ctypes
import hashlib
import io
import json
import math
import struct
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native
from .tensors import PrecisionMode, device_mode, precision_code

LN_EPS = 1e-6
TEXT_TABLE_ROWS = 1024
MODEL_MAGIC = b"DARTM1"
ROPE_BASE = 100.0


class ConfigError(ValueError):
    """A model configuration violates one of its invariants (model.py:33)."""


class MaskHeadRemovedError(RuntimeError):
    """Mask prediction was requested from a detection-only model (model.py:37)."""


@dataclass(frozen=True)
class ModelConfig:
    """Same fields, defaults and invariants as the reference (model.py:41-132)."""

    image_size: int = 64
    patch_size: int = 8
    embed_dim: int = 64
    num_blocks: int = 8
    global_block_indices: tuple[int, ...] = (3, 7)
    window_size: int = 4
    num_heads: int = 4
    fpn_dims: tuple[int, int, int] = (64, 64, 64)
    text_tokens: int = 8
    text_dim: int = 64
    num_queries: int = 16
    num_encoder_layers: int = 2
    num_decoder_layers: int = 2
    seed: int = 0

    @property
    def grid(self) -> int:
        return self.image_size // self.patch_size

    @property
    def tokens(self) -> int:
        return self.grid * self.grid

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.num_heads

    @property
    def mlp_hidden(self) -> int:
        return 4 * self.embed_dim

    @property
    def patch_dim(self) -> int:
        return self.patch_size * self.patch_size * 3

    def validate(self) -> None:
        if self.image_size <= 0 or self.patch_size <= 0:
            raise ConfigError("image_size and patch_size must be positive")
        if self.image_size % self.patch_size != 0:
            raise ConfigError(f"image_size {self.image_size} not divisible by patch_size {self.patch_size}")
        if self.grid % self.window_size != 0:
            raise ConfigError(f"token grid {self.grid} not divisible by window_size {self.window_size}")
        if self.grid % 4 != 0:
            raise ConfigError(f"token grid {self.grid} must be divisible by 4 for the 3 fpn levels")
        if self.num_blocks < 0:
            raise ConfigError("num_blocks must be non-negative")
        bad = [b for b in self.global_block_indices if not 0 <= b < self.num_blocks]
        if bad:
            raise ConfigError(f"global_block_indices {bad} outside [0, {self.num_blocks})")
        if self.num_blocks > 0 and not self.global_block_indices:
            raise ConfigError("at least one global block is required (sole cross-window path)")
        if self.embed_dim % self.num_heads != 0:
            raise ConfigError("embed_dim must divide evenly into num_heads")
        if self.head_dim % 4 != 0:
            raise ConfigError("head_dim must be divisible by 4 (2D rotary channel pairs)")
        if len(self.fpn_dims) != 3:
            raise ConfigError("fpn_dims must have exactly 3 entries")
        if self.text_dim % self.num_heads != 0:
            raise ConfigError("text_dim must divide evenly into num_heads")
        if min(self.text_tokens, self.num_queries, self.num_encoder_layers, self.num_decoder_layers) < 1:
            raise ConfigError("text_tokens, num_queries and layer counts must be >= 1")

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in self.__dataclass_fields__}
        d["global_block_indices"] = list(self.global_block_indices)
        d["fpn_dims"] = list(self.fpn_dims)
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "ModelConfig":
        d = dict(d)
        d["global_block_indices"] = tuple(d["global_block_indices"])
        d["fpn_dims"] = tuple(d["fpn_dims"])
        return cls(**d)


def toy_config(seed: int = 0, **overrides) -> ModelConfig:
    """The reference's desk-scale profile (model.py:135-137)."""
    return replace(ModelConfig(), seed=seed, **overrides)


def vit_h_config(seed: int = 0, **overrides) -> ModelConfig:
    """Full ViT-H/14 DART at 1008^2: 32 blocks (globals 7/15/23/31), 6+6 enc-dec,
    200 queries (BASELINE.json configs[1..4])."""
    base = ModelConfig(image_size=1008, patch_size=14, embed_dim=1280, num_blocks=32,
                       global_block_indices=(7, 15, 23, 31), window_size=24, num_heads=16,
                       fpn_dims=(256, 256, 256), text_tokens=32, text_dim=256, num_queries=200,
                       num_encoder_layers=6, num_decoder_layers=6, seed=seed)
    return replace(base, **overrides)


@dataclass
class DetectorModel:
    config: ModelConfig
    params: dict[str, np.ndarray]
    block_kinds: tuple[str, ...]
    attn_enabled: tuple[bool, ...]
    mlp_enabled: tuple[bool, ...]
    has_mask_head: bool = True
    plan_id: str | None = None
    _text_cache: dict[str, np.ndarray] = field(default_factory=dict, repr=False, compare=False)
    _handles: dict = field(default_factory=dict, repr=False, compare=False)
    _text_dev: dict = field(default_factory=dict, repr=False, compare=False)


class FpnFeatures:
    """Three class-agnostic feature levels plus provenance (model.py:152-166).

    The levels are GPU tensors (`device_levels`, float32 [T_l, F_l]) when produced by
    `backbone_forward`, or host arrays when a caller builds the record itself (the reference's
    distill.py:109-113 does); `.levels` is the reference-compatible float64 NumPy view, copied
    on first access.  Non-finite features raise ValueError at construction, as in the
    reference (the backbone's device-side finiteness flag is checked before it builds one)."""

    __slots__ = ("device_levels", "model_seed", "mode", "plan_id", "_host", "_l0_resident")

    def __init__(self, levels, model_seed: int, mode: PrecisionMode, plan_id: str | None = None,
                 l0_resident: bool = False, _finite_checked: bool = False):
        if len(levels) != 3:
            raise ValueError("fpn features must carry exactly 3 levels")
        levels = tuple(levels)
        on_device = [hasattr(t, "is_cuda") and t.is_cuda for t in levels]
        if not _finite_checked:
            for t, dev in zip(levels, on_device):
                finite = bool(t.isfinite().all().item()) if dev else bool(np.all(np.isfinite(np.asarray(t))))
                if not finite:
                    raise ValueError("fpn features must be finite")
        self.device_levels = levels
        self.model_seed = model_seed
        self.mode = mode
        self.plan_id = plan_id
        self._host = None
        self._l0_resident = l0_resident

    @property
    def levels(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        if self._host is None:
            self._host = tuple(
                t.detach().double().cpu().numpy() if hasattr(t, "detach") else np.asarray(t, dtype=np.float64)
                for t in self.device_levels)
        return self._host


@dataclass(frozen=True)
class TextEmbeddings:
    by_name: dict[str, np.ndarray]

    def stack(self, names: list[str]) -> list[np.ndarray]:
        return [self.by_name[n] for n in names]


class RawQueryOutputs:
    """Per-class decoder outputs before thresholding (model.py:177-188).  Device
    tensors (float64 boxes / logits, float32 query features) with lazy host views."""

    __slots__ = ("d_boxes", "d_score_logits", "d_presence_logits", "d_query_features", "_cache", "_batch")

    def __init__(self, d_boxes, d_score_logits, d_presence_logits, d_query_features=None):
        self.d_boxes = d_boxes
        self.d_score_logits = d_score_logits
        self.d_presence_logits = d_presence_logits
        self.d_query_features = d_query_features
        self._cache = {}
        self._batch = int(d_score_logits.shape[0])

    def _host(self, name, t):
        if name not in self._cache:
            self._cache[name] = None if t is None else t.detach().double().cpu().numpy()
        return self._cache[name]

    @property
    def boxes(self) -> np.ndarray:
        return self._host("boxes", self.d_boxes)

    @property
    def score_logits(self) -> np.ndarray:
        return self._host("score_logits", self.d_score_logits)

    @property
    def presence_logits(self) -> np.ndarray:
        return self._host("presence_logits", self.d_presence_logits)

    @property
    def query_features(self) -> np.ndarray | None:
        return self._host("query_features", self.d_query_features)

    @property
    def batch(self) -> int:
        return self._batch


# ---------------------------------------------------------------------------- init

def _philox_key(seed: int, path: str) -> int:
    """blake2b-128(seed␟path) little-endian (model.py:191-193)."""
    return int.from_bytes(hashlib.blake2b(f"{seed}\x1f{path}".encode(), digest_size=16).digest(), "little")


def _uniform_init(seed: int, path: str, shape, fan_in: int) -> np.ndarray:
    """U(-1, 1) / sqrt(fan_in) on the float32 grid (model.py:196-200)."""
    rng = np.random.Generator(np.random.Philox(key=_philox_key(seed, path)))
    return (rng.uniform(-1.0, 1.0, size=shape) / math.sqrt(fan_in)).astype(np.float32).astype(np.float64)


def _rope_tables(cfg: ModelConfig):
    """Row/column angles x 100^(-i/(hd/4)), cos/sin on the float32 grid (model.py:203-213)."""
    q = cfg.head_dim // 4
    inv = ROPE_BASE ** (-np.arange(q, dtype=np.float64) / q)
    r, c = np.divmod(np.arange(cfg.tokens, dtype=np.float64), float(cfg.grid))
    ang = np.concatenate([r[:, None] * inv[None, :], c[:, None] * inv[None, :]], axis=1)
    return np.cos(ang).astype(np.float32).astype(np.float64), np.sin(ang).astype(np.float32).astype(np.float64)


def param_declaration(cfg: ModelConfig, with_mask_head: bool) -> list[tuple[str, tuple, object]]:
    """Ordered (path, shape, init) list; the DARTM1 / C-ABI weight order (model.py:216-303)."""
    e, d, hid = cfg.embed_dim, cfg.text_dim, cfg.mlp_hidden
    decl = [("patch_embed.w", (cfg.patch_dim, e), cfg.patch_dim), ("patch_embed.b", (e,), "zeros"),
            ("rope.cos", (cfg.tokens, cfg.head_dim // 2), "rope_cos"),
            ("rope.sin", (cfg.tokens, cfg.head_dim // 2), "rope_sin")]
    for b in range(cfg.num_blocks):
        p = f"backbone.block{b}"
        decl += [(f"{p}.ln1.gamma", (e,), "ones"), (f"{p}.ln1.beta", (e,), "zeros"),
                 (f"{p}.attn.qkv.w", (e, 3 * e), e), (f"{p}.attn.qkv.b", (3 * e,), "zeros"),
                 (f"{p}.attn.out.w", (e, e), e), (f"{p}.attn.out.b", (e,), "zeros"),
                 (f"{p}.ln2.gamma", (e,), "ones"), (f"{p}.ln2.beta", (e,), "zeros"),
                 (f"{p}.mlp.fc1.w", (e, hid), e), (f"{p}.mlp.fc1.b", (hid,), "zeros"),
                 (f"{p}.mlp.fc2.w", (hid, e), hid), (f"{p}.mlp.fc2.b", (e,), "zeros")]
    for lvl in range(3):
        decl += [(f"fpn.level{lvl}.w", (e, cfg.fpn_dims[lvl]), e), (f"fpn.level{lvl}.b", (cfg.fpn_dims[lvl],), "zeros")]
    decl += [("text.table", (TEXT_TABLE_ROWS, d), 1), ("encdec.input.w", (cfg.fpn_dims[0], d), cfg.fpn_dims[0]),
             ("encdec.input.b", (d,), "zeros")]

    def ln(p):
        return [(f"{p}.gamma", (d,), "ones"), (f"{p}.beta", (d,), "zeros")]

    def attn(p):
        return [(f"{p}.q.w", (d, d), d), (f"{p}.q.b", (d,), "zeros"), (f"{p}.kv.w", (d, 2 * d), d),
                (f"{p}.kv.b", (2 * d,), "zeros"), (f"{p}.out.w", (d, d), d), (f"{p}.out.b", (d,), "zeros")]

    def mlp(p):
        return [(f"{p}.fc1.w", (d, 4 * d), d), (f"{p}.fc1.b", (4 * d,), "zeros"),
                (f"{p}.fc2.w", (4 * d, d), 4 * d), (f"{p}.fc2.b", (d,), "zeros")]

    def layer(p):
        return ln(f"{p}.ln1") + attn(f"{p}.self") + ln(f"{p}.ln2") + attn(f"{p}.cross") + ln(f"{p}.ln3") + mlp(f"{p}.mlp")

    for l in range(cfg.num_encoder_layers):
        decl += layer(f"encoder.layer{l}")
    decl += ln("encoder.final_ln")
    decl += [("decoder.queries", (cfg.num_queries, d), d), ("decoder.presence_token", (1, d), d)]
    for l in range(cfg.num_decoder_layers):
        decl += layer(f"decoder.layer{l}")
    decl += ln("decoder.final_ln")
    decl += [("heads.box.w", (d, 4), d), ("heads.box.b", (4,), "zeros"), ("heads.score.w", (d, 1), d),
             ("heads.score.b", (1,), "zeros"), ("heads.presence.w", (d, 1), d), ("heads.presence.b", (1,), "zeros")]
    if with_mask_head:
        decl += [("mask.query_proj.w", (d, d), d), ("mask.query_proj.b", (d,), "zeros"),
                 ("mask.feat_proj.w", (cfg.fpn_dims[0], d), cfg.fpn_dims[0]), ("mask.feat_proj.b", (d,), "zeros")]
    return decl


def build_model(config: ModelConfig, with_mask_head: bool = True) -> DetectorModel:
    """All weights from (seed, path), bit-identical to the reference (model.py:306-334)."""
    config.validate()
    cos, sin = _rope_tables(config)
    params: dict[str, np.ndarray] = {}
    for path, shape, init in param_declaration(config, with_mask_head):
        if init == "ones":
            params[path] = np.ones(shape)
        elif init == "zeros":
            params[path] = np.zeros(shape)
        elif init == "rope_cos":
            params[path] = cos
        elif init == "rope_sin":
            params[path] = sin
        else:
            params[path] = _uniform_init(config.seed, path, shape, int(init))
    kinds = tuple("global" if b in config.global_block_indices else "windowed" for b in range(config.num_blocks))
    on = tuple(True for _ in range(config.num_blocks))
    return DetectorModel(config=config, params=params, block_kinds=kinds, attn_enabled=on, mlp_enabled=on,
                         has_mask_head=with_mask_head)


def without_mask_head(model: DetectorModel) -> DetectorModel:
    params = {k: v for k, v in model.params.items() if not k.startswith("mask.")}
    return replace(model, params=params, has_mask_head=False, _handles={}, _text_dev={})


def sigmoid(x):
    """model.py:351-353."""
    return 1.0 / (1.0 + np.exp(-np.clip(x, -60.0, 60.0)))


# ---------------------------------------------------------------------------- device bridge

def _device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the DART B200 path needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_ptr(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


class _Handle:
    """One uploaded copy of a model's weights on one GPU (a `dart_model*`)."""

    def __init__(self, model: DetectorModel, device):
        import torch

        lib = _native.load()
        cfg = model.config
        desc = _native.ModelDesc()
        for k in ("image_size", "patch_size", "embed_dim", "num_blocks", "window_size", "num_heads", "text_tokens",
                  "text_dim", "num_queries", "num_encoder_layers", "num_decoder_layers"):
            setattr(desc, k, getattr(cfg, k))
        for i in range(3):
            desc.fpn_dims[i] = cfg.fpn_dims[i]
        if cfg.num_blocks > _native.MAX_BLOCKS:
            raise ValueError("too many blocks for the C ABI")
        for b in range(cfg.num_blocks):
            desc.block_global[b] = int(model.block_kinds[b] == "global")
            desc.attn_enabled[b] = int(model.attn_enabled[b])
            desc.mlp_enabled[b] = int(model.mlp_enabled[b])
        names = [p for p, _, _ in param_declaration(cfg, False)]
        missing = [n for n in names if n not in model.params]
        if missing:
            raise ValueError(f"model is missing parameters {missing[:3]}...")
        arrays = [np.ascontiguousarray(model.params[n], dtype=np.float32) for n in names]
        ptrs = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
        if lib.dart_expected_weight_count(ctypes.byref(desc)) != len(arrays):
            raise ValueError("parameter count does not match the C ABI's expectation")
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check(lib.dart_model_create(ctypes.byref(desc), ptrs, len(arrays), ctypes.byref(handle)))
            if model.has_mask_head and "mask.query_proj.w" in model.params:
                mk = [np.ascontiguousarray(model.params[n], dtype=np.float32)
                      for n in ("mask.query_proj.w", "mask.query_proj.b", "mask.feat_proj.w", "mask.feat_proj.b")]
                _native.check(lib.dart_model_set_mask_head(handle, *[a.ctypes.data for a in mk]))
        self.ptr = handle
        self.device = device
        self.lib = lib
        self.cfg = cfg

    def fork(self) -> "_Handle":
        """A second handle on the same device weights with its own activation workspace
        (dart_model_fork), for a second concurrent stream."""
        import torch

        f = object.__new__(_Handle)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.dart_model_fork(self.ptr, ctypes.byref(handle)))
        f.ptr, f.device, f.lib, f.cfg = handle, self.device, self.lib, self.cfg
        return f

    def __del__(self):
        try:
            if self.ptr:
                self.lib.dart_model_destroy(self.ptr)
        except Exception:
            pass


def native_handle(model: DetectorModel, device=None) -> _Handle:
    device = device or _device()
    key = (device.index, model.block_kinds, model.attn_enabled, model.mlp_enabled)
    h = model._handles.get(key)
    if h is None:
        h = _Handle(model, device)
        model._handles[key] = h
    return h


# ---------------------------------------------------------------------------- forwards

def _check_image(cfg: ModelConfig, image: np.ndarray) -> np.ndarray:
    image = np.asarray(image)
    expected = (cfg.image_size, cfg.image_size, 3)
    if image.shape[-3:] != expected or image.ndim not in (3, 4):
        raise ValueError(f"image shape {image.shape} does not match {expected}")
    return image


def backbone_forward_batch(model: DetectorModel, images, mode: PrecisionMode = PrecisionMode.FP32,
                           check: bool = True):
    """[B, S, S, 3] (NumPy or torch, host or device) -> device (L0, L1, L2) [B, T_l, F_l] and
    the device status flags.  `check=True` synchronises and raises like the reference."""
    import torch

    code = precision_code(mode)
    cfg = model.config
    dev = _device()
    h = native_handle(model, dev)
    if isinstance(images, torch.Tensor):
        imgs = images.to(device=dev, dtype=torch.float32).contiguous()
    else:
        imgs = torch.from_numpy(np.ascontiguousarray(_check_image(cfg, images), dtype=np.float32)).to(dev)
    if imgs.ndim == 3:
        imgs = imgs.unsqueeze(0)
    if tuple(imgs.shape[1:]) != (cfg.image_size, cfg.image_size, 3):
        raise ValueError(f"image shape {tuple(imgs.shape)} does not match {(cfg.image_size, cfg.image_size, 3)}")
    B = imgs.shape[0]
    T, g = cfg.tokens, cfg.grid
    l0 = torch.empty((B, T, cfg.fpn_dims[0]), device=dev, dtype=torch.float32)
    l1 = torch.empty((B, (g // 2) ** 2, cfg.fpn_dims[1]), device=dev, dtype=torch.float32)
    l2 = torch.empty((B, (g // 4) ** 2, cfg.fpn_dims[2]), device=dev, dtype=torch.float32)
    flags = torch.zeros((1,), device=dev, dtype=torch.int32)
    _native.check(h.lib.dart_model_set_precision(h.ptr, code))
    try:
        _native.check(h.lib.dart_backbone(h.ptr, imgs.data_ptr(), B, l0.data_ptr(), l1.data_ptr(), l2.data_ptr(),
                                          flags.data_ptr(), _stream_ptr(dev)))
    finally:
        _native.check(h.lib.dart_model_set_precision(h.ptr, 0))
    if check:
        raise_for_flags(int(flags.item()))
    return (l0, l1, l2), flags


def raise_for_flags(f: int) -> None:
    if f & _native.FLAG_IMAGE_RANGE:
        raise ValueError("image values must lie in [0, 1]")
    if f & _native.FLAG_NONFINITE:
        raise ValueError("fpn features must be finite")


def backbone_forward(model: DetectorModel, image: np.ndarray, mode: PrecisionMode = PrecisionMode.FP32) -> FpnFeatures:
    """Image -> 3-level feature pyramid on the GPU (model.py:454-459).  Text never enters."""
    image = _check_image(model.config, image)
    if image.ndim != 3:
        raise ValueError(f"image shape {image.shape} does not match {(model.config.image_size,) * 2 + (3,)}")
    (l0, l1, l2), _ = backbone_forward_batch(model, image, mode)  # raises on the device flags
    return FpnFeatures((l0[0], l1[0], l2[0]), model.config.seed, device_mode(mode, backbone=True), model.plan_id,
                       _finite_checked=True)


def _text_rows(name: str, text_tokens: int) -> list[int]:
    """blake2b-64(name␟i) mod 1024 (model.py:462-467)."""
    return [int.from_bytes(hashlib.blake2b(f"{name}\x1f{i}".encode(), digest_size=8).digest(), "little")
            % TEXT_TABLE_ROWS for i in range(text_tokens)]


def text_encode(model: DetectorModel, class_names: list[str]) -> TextEmbeddings:
    """Hash each class name into embedding-table rows; memoised per model (model.py:470-484)."""
    if not class_names:
        raise ValueError("class name list is empty")
    out: dict[str, np.ndarray] = {}
    for name in class_names:
        if not name:
            raise ValueError("class names must be non-empty strings")
        if name not in model._text_cache:
            emb = model.params["text.table"][_text_rows(name, model.config.text_tokens)].copy()
            emb.setflags(write=False)
            model._text_cache[name] = emb
        out[name] = model._text_cache[name]
    return TextEmbeddings(out)


def clear_text_cache(model: DetectorModel) -> None:
    model._text_cache.clear()
    model._text_dev.clear()


def device_text(model: DetectorModel, text_batch: list[np.ndarray], dev):
    """[N, L_t, d] float32 device tensor; rows served from the per-model device cache when
    the arrays are the cached embeddings (the K15 'text-embedding gather to device')."""
    import torch

    rows = []
    for t in text_batch:
        key = id(t)
        hit = model._text_dev.get(key)
        if hit is not None and hit[0] is t:
            rows.append(hit[1])
            continue
        d = torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32)).to(dev)
        if not t.flags.writeable:  # cached, immutable embedding
            model._text_dev[key] = (t, d)
        rows.append(d)
    return torch.stack(rows)


def _validate_text(cfg: ModelConfig, text_batch) -> None:
    if len(text_batch) < 1:
        raise ValueError("text batch must contain at least one class")
    for t in text_batch:
        if tuple(np.shape(t)) != (cfg.text_tokens, cfg.text_dim):
            raise ValueError(f"text embedding shape {np.shape(t)} does not match model")


def encdec_forward_device(model: DetectorModel, l0, text, B: int, N: int, with_query_features: bool = True,
                          reuse_backbone: bool = False):
    """Device-level class-batched enc-dec: l0 [B, T, F0] f32 (or None when reuse_backbone),
    text [N, L_t, d] f32 -> RawQueryOutputs over B*N items (item = b*N + c)."""
    import torch

    cfg = model.config
    dev = _device()
    h = native_handle(model, dev)
    items = B * N
    Q = cfg.num_queries
    boxes = torch.empty((items, Q, 4), device=dev, dtype=torch.float64)
    scores = torch.empty((items, Q), device=dev, dtype=torch.float64)
    pres = torch.empty((items,), device=dev, dtype=torch.float64)
    qf = torch.empty((items, Q, cfg.text_dim), device=dev, dtype=torch.float32) if with_query_features else None
    l0p = None if reuse_backbone else l0.contiguous().data_ptr()
    _native.check(h.lib.dart_encdec(h.ptr, l0p, B, text.contiguous().data_ptr(), N, boxes.data_ptr(),
                                    scores.data_ptr(), pres.data_ptr(), qf.data_ptr() if qf is not None else None,
                                    _stream_ptr(dev)))
    return RawQueryOutputs(boxes, scores, pres, qf)


def encdec_forward(model: DetectorModel, fpn: FpnFeatures, text_batch: list[np.ndarray],
                   mode: PrecisionMode = PrecisionMode.FP32) -> RawQueryOutputs:
    """Decode a batch of class prompts against shared image features (model.py:536-570):
    one class-batched pass on the GPU, classes independent by construction."""
    import torch

    device_mode(mode)
    cfg = model.config
    _validate_text(cfg, text_batch)
    if isinstance(fpn, FpnFeatures):
        l0 = fpn.device_levels[0]
    else:
        l0 = fpn.levels[0]
    if tuple(l0.shape) != (cfg.tokens, cfg.fpn_dims[0]):
        raise ValueError(f"fpn level-0 shape {tuple(l0.shape)} does not match model {(cfg.tokens, cfg.fpn_dims[0])}")
    dev = _device()
    if not isinstance(l0, torch.Tensor):
        l0 = torch.from_numpy(np.ascontiguousarray(l0, dtype=np.float32))
    l0 = l0.to(device=dev, dtype=torch.float32).reshape(1, cfg.tokens, cfg.fpn_dims[0])
    text = device_text(model, text_batch, dev)
    return encdec_forward_device(model, l0, text, 1, len(text_batch))


def mask_head_forward_device(model: DetectorModel, l0, query_features, B: int = 1):
    """Device mask logits: l0 [B, T, F0] f32, query_features [B*N, Q, d] f32 (torch, cuda) ->
    [B*N, Q, T] f32 = (qf Wq + bq)(L0[b] Wf + bf)^T (model.py:573-579)."""
    import torch

    if not model.has_mask_head:
        raise MaskHeadRemovedError("mask head removed: this model is detection-only")
    cfg = model.config
    dev = _device()
    h = native_handle(model, dev)
    items = int(query_features.shape[0])
    if items % B:
        raise ValueError("query feature batch is not a multiple of the image batch")
    out = torch.empty((items, cfg.num_queries, cfg.tokens), device=dev, dtype=torch.float32)
    _native.check(h.lib.dart_mask_head(h.ptr, query_features.contiguous().data_ptr(), B, items // B,
                                       l0.contiguous().data_ptr(), out.data_ptr(), _stream_ptr(dev)))
    return out


def mask_head_forward(model: DetectorModel, fpn: FpnFeatures, queries: RawQueryOutputs) -> np.ndarray:
    """Per-query mask logits over the level-0 token grid [N, queries, tokens] (model.py:573-579),
    computed on the GPU (fp16 operands, fp32 accumulation); float64 host array like the reference."""
    import torch

    if not model.has_mask_head:
        raise MaskHeadRemovedError("mask head removed: this model is detection-only")
    cfg = model.config
    dev = _device()
    l0 = fpn.device_levels[0] if isinstance(fpn, FpnFeatures) else torch.from_numpy(
        np.ascontiguousarray(fpn.levels[0], dtype=np.float32))
    l0 = l0.to(device=dev, dtype=torch.float32).reshape(1, cfg.tokens, cfg.fpn_dims[0])
    qf = getattr(queries, "d_query_features", None)
    if qf is None:
        qf = torch.from_numpy(np.ascontiguousarray(queries.query_features, dtype=np.float32))
    qf = qf.to(device=dev, dtype=torch.float32)
    return mask_head_forward_device(model, l0, qf, 1).double().cpu().numpy()


# ---------------------------------------------------------------------------- structural edits

def set_sub_block(model: DetectorModel, block: int, kind: str, enabled: bool) -> DetectorModel:
    """model.py:587-595."""
    if kind not in ("attn", "mlp"):
        raise ValueError(f"unknown sub-block kind {kind!r}")
    if not 0 <= block < model.config.num_blocks:
        raise ValueError(f"block index {block} out of range")
    attn, mlp = list(model.attn_enabled), list(model.mlp_enabled)
    (attn if kind == "attn" else mlp)[block] = enabled
    return replace(model, attn_enabled=tuple(attn), mlp_enabled=tuple(mlp), _handles={}, _text_dev={})


def truncate_model(model: DetectorModel, depth: int) -> DetectorModel:
    """Keep the first `depth` blocks; re-tag the last one global if none survives (model.py:598-625)."""
    cfg = model.config
    if not 0 <= depth <= cfg.num_blocks:
        raise ValueError(f"depth {depth} exceeds num_blocks {cfg.num_blocks}")
    kept_globals = tuple(b for b in cfg.global_block_indices if b < depth)
    kinds = list(model.block_kinds[:depth])
    if depth > 0 and not kept_globals:
        kinds[depth - 1] = "global"
        kept_globals = (depth - 1,)
    params = {k: v for k, v in model.params.items()
              if not k.startswith("backbone.block") or int(k.split(".")[1][5:]) < depth}
    return replace(model, config=replace(cfg, num_blocks=depth, global_block_indices=kept_globals), params=params,
                   block_kinds=tuple(kinds), attn_enabled=model.attn_enabled[:depth],
                   mlp_enabled=model.mlp_enabled[:depth], _handles={}, _text_dev={})


# ---------------------------------------------------------------------------- serialization

def save_model(model: DetectorModel, path) -> None:
    """DARTM1: magic, u32 header length, canonical JSON header, float32 LE weights in
    declaration order (model.py:633-654)."""
    names = list(model.params.keys())
    header = {"config": model.config.to_dict(), "block_kinds": list(model.block_kinds),
              "attn_enabled": list(model.attn_enabled), "mlp_enabled": list(model.mlp_enabled),
              "has_mask_head": model.has_mask_head, "plan_id": model.plan_id,
              "params": [[n, list(model.params[n].shape)] for n in names]}
    blob = json.dumps(header, sort_keys=True, separators=(",", ":")).encode("utf-8")
    buf = io.BytesIO()
    buf.write(MODEL_MAGIC)
    buf.write(struct.pack("<I", len(blob)))
    buf.write(blob)
    for n in names:
        buf.write(model.params[n].astype("<f4").tobytes())
    with open(path, "wb") as f:
        f.write(buf.getvalue())


def load_model(path) -> DetectorModel:
    """model.py:657-681."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[: len(MODEL_MAGIC)] != MODEL_MAGIC:
        raise ValueError("not a model file (bad magic)")
    off = len(MODEL_MAGIC)
    (hlen,) = struct.unpack_from("<I", raw, off)
    off += 4
    header = json.loads(raw[off: off + hlen].decode("utf-8"))
    off += hlen
    params = {}
    for name, shape in header["params"]:
        count = int(np.prod(shape)) if shape else 1
        params[name] = np.frombuffer(raw, dtype="<f4", count=count, offset=off).astype(np.float64).reshape(shape)
        off += 4 * count
    return DetectorModel(config=ModelConfig.from_dict(header["config"]), params=params,
                         block_kinds=tuple(header["block_kinds"]), attn_enabled=tuple(header["attn_enabled"]),
                         mlp_enabled=tuple(header["mlp_enabled"]), has_mask_head=header["has_mask_head"],
                         plan_id=header["plan_id"])


def models_equal(a: DetectorModel, b: DetectorModel) -> bool:
    if a.config != b.config or a.block_kinds != b.block_kinds:
        return False
    if a.attn_enabled != b.attn_enabled or a.mlp_enabled != b.mlp_enabled:
        return False
    if a.params.keys() != b.params.keys():
        return False
    return all(np.array_equal(a.params[k], b.params[k]) for k in a.params)


def weights_checksum(model: DetectorModel, prefixes: tuple[str, ...] = ()) -> str:
    """blake2b-128 over (name, float64 bytes) (model.py:694-702)."""
    h = hashlib.blake2b(digest_size=16)
    for name in model.params:
        if prefixes and not name.startswith(prefixes):
            continue
        h.update(name.encode())
        h.update(model.params[name].tobytes())
    return h.hexdigest()


ENCDEC_PREFIXES = ("encdec.", "encoder.", "decoder.", "heads.")
