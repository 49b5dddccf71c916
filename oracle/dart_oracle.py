"""CPU oracle for DART's multi-class detection path -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference algorithm
(`/root/reference/pkg/src/dart/{model,pipeline,scenes,tensors}.py`), written
from its documented behaviour.  It is the checker for the B200 path: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product package
(`paper_2603_11441_b200`) never imports it and has no CPU fallback.

Parity pinning: `oracle/make_golden.py` runs the real reference in the build
container and writes `tests/golden/*.npz`; `tests/test_oracle.py` checks this
restatement against those fixtures (weights bit-exact, activations and raw
outputs to ~1e-10 relative, detections exactly).

Every function cites the reference file:line it restates.  Arithmetic is the
reference's `PrecisionMode.FP32` discipline (plain float64, `tensors.py:164-165,
194-197`); the half-precision emulation modes are out of scope.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

LN_EPS = 1e-6            # model.py:27
TEXT_TABLE_ROWS = 1024   # model.py:28
ROPE_BASE = 100.0        # model.py:30


@dataclass(frozen=True)
class OracleConfig:
    """Dimensions of the detector (model.py:41-76)."""

    image_size: int = 64
    patch_size: int = 8
    embed_dim: int = 64
    num_blocks: int = 8
    global_block_indices: tuple = (3, 7)
    window_size: int = 4
    num_heads: int = 4
    fpn_dims: tuple = (64, 64, 64)
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


def full_config(seed: int = 0, **over) -> OracleConfig:
    """ViT-H/14 DART at 1008^2."""
    base = dict(image_size=1008, patch_size=14, embed_dim=1280, num_blocks=32,
                global_block_indices=(7, 15, 23, 31), window_size=24, num_heads=16,
                fpn_dims=(256, 256, 256), text_tokens=32, text_dim=256, num_queries=200,
                num_encoder_layers=6, num_decoder_layers=6, seed=seed)
    base.update(over)
    return OracleConfig(**base)


def small1008_config(seed: int = 0) -> OracleConfig:
    """Config B of SURVEY.md 8(d): full width, 4 blocks, 6+6 enc-dec."""
    return full_config(seed, num_blocks=4, global_block_indices=(1, 3))


# ----------------------------------------------------------------------------
# deterministic weights (model.py:191-334)
# ----------------------------------------------------------------------------

def philox_uniform(seed: int, path: str, shape, fan_in: int) -> np.ndarray:
    """U(-1,1)/sqrt(fan_in) from Philox keyed by blake2b(seed␟path), float32 grid
    (model.py:191-200)."""
    key = int.from_bytes(hashlib.blake2b(f"{seed}\x1f{path}".encode(), digest_size=16).digest(), "little")
    rng = np.random.Generator(np.random.Philox(key=key))
    return (rng.uniform(-1.0, 1.0, size=shape) / math.sqrt(fan_in)).astype(np.float32).astype(np.float64)


def rope_tables(cfg: OracleConfig):
    """Per-token (row, col) angles times 100^(-i/(hd/4)), cos/sin snapped to float32
    (model.py:203-213)."""
    quarter = cfg.head_dim // 4
    inv = ROPE_BASE ** (-np.arange(quarter, dtype=np.float64) / quarter)
    t = np.arange(cfg.tokens, dtype=np.float64)
    r, c = np.floor(t / cfg.grid), np.mod(t, cfg.grid)
    ang = np.concatenate([np.outer(r, inv), np.outer(c, inv)], axis=1)
    return (np.cos(ang).astype(np.float32).astype(np.float64),
            np.sin(ang).astype(np.float32).astype(np.float64))


def param_declaration(cfg: OracleConfig, with_mask_head: bool = False):
    """Ordered (path, shape, init) list (model.py:216-303)."""
    e, d, hid = cfg.embed_dim, cfg.text_dim, 4 * cfg.embed_dim
    out = [("patch_embed.w", (3 * cfg.patch_size ** 2, e), 3 * cfg.patch_size ** 2),
           ("patch_embed.b", (e,), "zeros"),
           ("rope.cos", (cfg.tokens, cfg.head_dim // 2), "rope_cos"),
           ("rope.sin", (cfg.tokens, cfg.head_dim // 2), "rope_sin")]
    for b in range(cfg.num_blocks):
        p = f"backbone.block{b}"
        out += [(f"{p}.ln1.gamma", (e,), "ones"), (f"{p}.ln1.beta", (e,), "zeros"),
                (f"{p}.attn.qkv.w", (e, 3 * e), e), (f"{p}.attn.qkv.b", (3 * e,), "zeros"),
                (f"{p}.attn.out.w", (e, e), e), (f"{p}.attn.out.b", (e,), "zeros"),
                (f"{p}.ln2.gamma", (e,), "ones"), (f"{p}.ln2.beta", (e,), "zeros"),
                (f"{p}.mlp.fc1.w", (e, hid), e), (f"{p}.mlp.fc1.b", (hid,), "zeros"),
                (f"{p}.mlp.fc2.w", (hid, e), hid), (f"{p}.mlp.fc2.b", (e,), "zeros")]
    for lvl in range(3):
        out += [(f"fpn.level{lvl}.w", (e, cfg.fpn_dims[lvl]), e),
                (f"fpn.level{lvl}.b", (cfg.fpn_dims[lvl],), "zeros")]
    out += [("text.table", (TEXT_TABLE_ROWS, d), 1),
            ("encdec.input.w", (cfg.fpn_dims[0], d), cfg.fpn_dims[0]),
            ("encdec.input.b", (d,), "zeros")]

    def ln(p):
        return [(f"{p}.gamma", (d,), "ones"), (f"{p}.beta", (d,), "zeros")]

    def attn(p):
        return [(f"{p}.q.w", (d, d), d), (f"{p}.q.b", (d,), "zeros"),
                (f"{p}.kv.w", (d, 2 * d), d), (f"{p}.kv.b", (2 * d,), "zeros"),
                (f"{p}.out.w", (d, d), d), (f"{p}.out.b", (d,), "zeros")]

    def mlp(p):
        return [(f"{p}.fc1.w", (d, 4 * d), d), (f"{p}.fc1.b", (4 * d,), "zeros"),
                (f"{p}.fc2.w", (4 * d, d), 4 * d), (f"{p}.fc2.b", (d,), "zeros")]

    for stack, n in (("encoder", cfg.num_encoder_layers),):
        for l in range(n):
            p = f"{stack}.layer{l}"
            out += ln(f"{p}.ln1") + attn(f"{p}.self") + ln(f"{p}.ln2") + attn(f"{p}.cross") + ln(f"{p}.ln3") + mlp(f"{p}.mlp")
    out += ln("encoder.final_ln")
    out += [("decoder.queries", (cfg.num_queries, d), d), ("decoder.presence_token", (1, d), d)]
    for l in range(cfg.num_decoder_layers):
        p = f"decoder.layer{l}"
        out += ln(f"{p}.ln1") + attn(f"{p}.self") + ln(f"{p}.ln2") + attn(f"{p}.cross") + ln(f"{p}.ln3") + mlp(f"{p}.mlp")
    out += ln("decoder.final_ln")
    out += [("heads.box.w", (d, 4), d), ("heads.box.b", (4,), "zeros"),
            ("heads.score.w", (d, 1), d), ("heads.score.b", (1,), "zeros"),
            ("heads.presence.w", (d, 1), d), ("heads.presence.b", (1,), "zeros")]
    if with_mask_head:
        out += [("mask.query_proj.w", (d, d), d), ("mask.query_proj.b", (d,), "zeros"),
                ("mask.feat_proj.w", (cfg.fpn_dims[0], d), cfg.fpn_dims[0]),
                ("mask.feat_proj.b", (d,), "zeros")]
    return out


def build_params(cfg: OracleConfig, with_mask_head: bool = False) -> dict:
    """model.py:306-334."""
    cos, sin = rope_tables(cfg)
    params = {}
    for path, shape, init in param_declaration(cfg, with_mask_head):
        if init == "ones":
            params[path] = np.ones(shape)
        elif init == "zeros":
            params[path] = np.zeros(shape)
        elif init == "rope_cos":
            params[path] = cos
        elif init == "rope_sin":
            params[path] = sin
        else:
            params[path] = philox_uniform(cfg.seed, path, shape, int(init))
    return params


def weights_checksum(params: dict, order=None) -> str:
    """blake2b-128 over (name, float64 bytes) in declaration order (model.py:694-702)."""
    h = hashlib.blake2b(digest_size=16)
    for name in (order or params.keys()):
        h.update(name.encode())
        h.update(np.ascontiguousarray(params[name], dtype=np.float64).tobytes())
    return h.hexdigest()


# ----------------------------------------------------------------------------
# float64 primitives (tensors.py)
# ----------------------------------------------------------------------------

def sigmoid(x):
    """model.py:351-353."""
    return 1.0 / (1.0 + np.exp(-np.clip(x, -60.0, 60.0)))


def layernorm(x, g, b):
    """Population variance, eps 1e-6 (tensors.py:215-227)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * g + b


def softmax_last(s):
    """Max-subtracted softmax over the last axis (tensors.py:194-197)."""
    z = np.exp(s - s.max(axis=-1, keepdims=True))
    return z / z.sum(axis=-1, keepdims=True)


def rope(x, cos, sin):
    """Rotate interleaved channel pairs (2j, 2j+1) by tabulated angles
    (tensors.py:235-252).  x: [..., T, hd]; tables [T, hd/2]."""
    ev, od = x[..., 0::2], x[..., 1::2]
    y = np.empty_like(x)
    y[..., 0::2] = ev * cos - od * sin
    y[..., 1::2] = ev * sin + od * cos
    return y


def linear(P, x, path):
    """y = x @ W + b with W stored [in, out] (model.py:356-358)."""
    return x @ P[f"{path}.w"] + P[f"{path}.b"]


def sdpa(q, k, v):
    """softmax(q k^T / sqrt(hd)) v over [..., L, hd] (model.py:403-406, 498-501)."""
    s = (q @ np.swapaxes(k, -1, -2)) / math.sqrt(q.shape[-1])
    return softmax_last(s) @ v


# ----------------------------------------------------------------------------
# backbone (model.py:375-459)
# ----------------------------------------------------------------------------

def patchify(cfg: OracleConfig, image: np.ndarray) -> np.ndarray:
    """[S,S,3] -> [T, p*p*3], token t = r*grid + c, patch order (py, px, ch)
    (model.py:426-436).  Validates shape and the [0, 1] range."""
    image = np.asarray(image, dtype=np.float64)
    if image.shape != (cfg.image_size, cfg.image_size, 3):
        raise ValueError(f"image shape {image.shape} does not match {(cfg.image_size, cfg.image_size, 3)}")
    if image.min() < 0.0 or image.max() > 1.0:
        raise ValueError("image values must lie in [0, 1]")
    g, p = cfg.grid, cfg.patch_size
    return image.reshape(g, p, g, p, 3).swapaxes(1, 2).reshape(g * g, p * p * 3)


def window_token_order(cfg: OracleConfig) -> np.ndarray:
    """Permutation listing tokens window by window (window id (r//w)*(g/w)+(c//w),
    in-window index (r%w)*w + (c%w); model.py:375-387)."""
    g, w = cfg.grid, cfg.window_size
    n = g // w
    idx = np.arange(g * g).reshape(n, w, n, w).transpose(0, 2, 1, 3)
    return idx.reshape(-1)


def block_attention(P, cfg: OracleConfig, h, b: int, windowed: bool):
    """model.py:390-409."""
    T, H, hd = cfg.tokens, cfg.num_heads, cfg.head_dim
    qkv = linear(P, h, f"backbone.block{b}.attn.qkv").reshape(T, 3, H, hd)
    q, k, v = (np.ascontiguousarray(qkv[:, i].transpose(1, 0, 2)) for i in range(3))
    q = rope(q, P["rope.cos"], P["rope.sin"])
    k = rope(k, P["rope.cos"], P["rope.sin"])
    if windowed:
        order = window_token_order(cfg)
        nw, wl = (cfg.grid // cfg.window_size) ** 2, cfg.window_size ** 2
        qw, kw, vw = (a[:, order].reshape(H, nw, wl, hd) for a in (q, k, v))
        ow = sdpa(qw, kw, vw).reshape(H, T, hd)
        o = np.empty_like(ow)
        o[:, order] = ow
    else:
        o = sdpa(q, k, v)
    return linear(P, o.transpose(1, 0, 2).reshape(T, H * hd), f"backbone.block{b}.attn.out")


def backbone_block(P, cfg: OracleConfig, x, b: int, attn_on=True, mlp_on=True):
    """Pre-LN residual block with ReLU MLP (model.py:412-423)."""
    pre = f"backbone.block{b}"
    if attn_on:
        x = x + block_attention(P, cfg, layernorm(x, P[f"{pre}.ln1.gamma"], P[f"{pre}.ln1.beta"]), b,
                                b not in cfg.global_block_indices)
    if mlp_on:
        h = layernorm(x, P[f"{pre}.ln2.gamma"], P[f"{pre}.ln2.beta"])
        h = np.maximum(linear(P, h, f"{pre}.mlp.fc1"), 0.0)
        x = x + linear(P, h, f"{pre}.mlp.fc2")
    return x


def pool(cfg: OracleConfig, x, f: int):
    """Mean over f x f token blocks (model.py:439-443)."""
    g = cfg.grid // f
    return x.reshape(g, f, g, f, x.shape[-1]).mean(axis=(1, 3)).reshape(g * g, x.shape[-1])


def fpn(P, cfg: OracleConfig, x):
    """model.py:446-451."""
    return (linear(P, x, "fpn.level0"), linear(P, pool(cfg, x, 2), "fpn.level1"),
            linear(P, pool(cfg, x, 4), "fpn.level2"))


def backbone(P, cfg: OracleConfig, image, taps: dict | None = None, attn_on=None, mlp_on=None):
    """image -> (L0, L1, L2) (model.py:454-459).  `taps` collects the residual
    stream after patch-embed ('tokens') and after every block ('block{b}')."""
    x = linear(P, patchify(cfg, image), "patch_embed")
    if taps is not None:
        taps["tokens"] = x
    for b in range(cfg.num_blocks):
        x = backbone_block(P, cfg, x, b, True if attn_on is None else attn_on[b],
                           True if mlp_on is None else mlp_on[b])
        if taps is not None:
            taps[f"block{b}"] = x
    levels = fpn(P, cfg, x)
    for lvl in levels:
        if not np.all(np.isfinite(lvl)):
            raise ValueError("fpn features must be finite")
    return levels


# ----------------------------------------------------------------------------
# text + enc-dec (model.py:462-570)
# ----------------------------------------------------------------------------

def text_rows(name: str, n: int):
    """blake2b-64(name␟i) mod 1024 (model.py:462-467)."""
    return [int.from_bytes(hashlib.blake2b(f"{name}\x1f{i}".encode(), digest_size=8).digest(), "little")
            % TEXT_TABLE_ROWS for i in range(n)]


def text_embedding(P, cfg: OracleConfig, name: str):
    if not name:
        raise ValueError("class names must be non-empty strings")
    return P["text.table"][text_rows(name, cfg.text_tokens)]


def mha(P, cfg: OracleConfig, x_q, x_kv, prefix: str):
    """Multi-head attention with contiguous d/H head chunks (model.py:491-502)."""
    H, d = cfg.num_heads, cfg.text_dim
    dh = d // H
    q = linear(P, x_q, f"{prefix}.q")
    kv = linear(P, x_kv, f"{prefix}.kv")
    split = lambda a: a.reshape(a.shape[0], H, dh).transpose(1, 0, 2)
    o = sdpa(split(q), split(kv[:, :d]), split(kv[:, d:]))
    return linear(P, o.transpose(1, 0, 2).reshape(-1, d), f"{prefix}.out")


def mlp(P, x, prefix: str):
    """model.py:505-508."""
    return linear(P, np.maximum(linear(P, x, f"{prefix}.fc1"), 0.0), f"{prefix}.fc2")


def _ln(P, x, p):
    return layernorm(x, P[f"{p}.gamma"], P[f"{p}.beta"])


def encoder_prefix(P, cfg: OracleConfig, level0):
    """Class-independent part: input projection and encoder layer-0 self-attention
    (model.py:513-517 up to the first text use)."""
    e = linear(P, level0, "encdec.input")
    h = _ln(P, e, "encoder.layer0.ln1")
    return e + mha(P, cfg, h, h, "encoder.layer0.self")


def encdec_one(P, cfg: OracleConfig, level0, text, taps: dict | None = None, e1=None):
    """One class: 6-layer encoder, 6-layer decoder, heads (model.py:511-533).
    Returns (query_features, boxes, presence_logit, score_logits).  `e1`: the class-independent
    prefix output (encoder_prefix) when already computed; level0 is then unused."""
    e = encoder_prefix(P, cfg, level0) if e1 is None else e1
    for l in range(cfg.num_encoder_layers):
        p = f"encoder.layer{l}"
        if l > 0:
            h = _ln(P, e, f"{p}.ln1")
            e = e + mha(P, cfg, h, h, f"{p}.self")
        e = e + mha(P, cfg, _ln(P, e, f"{p}.ln2"), text, f"{p}.cross")
        e = e + mlp(P, _ln(P, e, f"{p}.ln3"), f"{p}.mlp")
        if taps is not None:
            taps[f"enc{l}"] = e
    mem = _ln(P, e, "encoder.final_ln")
    if taps is not None:
        taps["memory"] = mem
    q = np.concatenate([P["decoder.queries"], P["decoder.presence_token"]], axis=0)
    for l in range(cfg.num_decoder_layers):
        p = f"decoder.layer{l}"
        h = _ln(P, q, f"{p}.ln1")
        q = q + mha(P, cfg, h, h, f"{p}.self")
        q = q + mha(P, cfg, _ln(P, q, f"{p}.ln2"), mem, f"{p}.cross")
        q = q + mlp(P, _ln(P, q, f"{p}.ln3"), f"{p}.mlp")
        if taps is not None:
            taps[f"dec{l}"] = q
    q = _ln(P, q, "decoder.final_ln")
    nq = cfg.num_queries
    qf = q[:nq]
    boxes = sigmoid(linear(P, qf, "heads.box"))
    scores = linear(P, qf, "heads.score")[:, 0]
    presence = float(linear(P, q[nq:], "heads.presence")[0, 0])
    return qf, boxes, presence, scores


def encdec(P, cfg: OracleConfig, level0, texts, e1=None):
    """Classes decoded independently and stacked (model.py:536-570)."""
    if len(texts) < 1:
        raise ValueError("text batch must contain at least one class")
    outs = [encdec_one(P, cfg, level0, t, e1=e1) for t in texts]
    return (np.stack([o[0] for o in outs]), np.stack([o[1] for o in outs]),
            np.array([o[2] for o in outs], dtype=np.float64), np.stack([o[3] for o in outs]))


def mask_head(P, level0, query_features):
    """Per-query mask logits over the level-0 grid (model.py:573-579):
    (qf Wq + bq) (L0 Wf + bf)^T -> [N, queries, tokens]."""
    mq = query_features @ P["mask.query_proj.w"] + P["mask.query_proj.b"]
    mf = level0 @ P["mask.feat_proj.w"] + P["mask.feat_proj.b"]
    return mq @ mf.T


# ----------------------------------------------------------------------------
# post-processing (pipeline.py:243-294)
# ----------------------------------------------------------------------------

def box_iou(a, b) -> float:
    """(cx, cy, w, h) IoU, corners computed the reference's way (pipeline.py:243-254)."""
    ax0, ax1 = a[0] - a[2] / 2, a[0] + a[2] / 2
    ay0, ay1 = a[1] - a[3] / 2, a[1] + a[3] / 2
    bx0, bx1 = b[0] - b[2] / 2, b[0] + b[2] / 2
    by0, by1 = b[1] - b[3] / 2, b[1] + b[3] / 2
    iw = min(ax1, bx1) - max(ax0, bx0)
    ih = min(ay1, by1) - max(ay0, by0)
    if iw <= 0.0 or ih <= 0.0:
        return 0.0
    inter = iw * ih
    return inter / (a[2] * a[3] + b[2] * b[3] - inter)


def greedy_nms(cands, thr: float):
    """Keep a candidate iff its IoU with every kept one is < thr (pipeline.py:257-263)."""
    kept = []
    for c in cands:
        if all(box_iou(c[0], k[0]) < thr for k in kept):
            kept.append(c)
    return kept


def postprocess(boxes, score_logits, presence_logits, presence_thr=0.5, score_thr=0.45,
                nms_thr=0.5, cross_class=False):
    """Presence gate, score gate, (score desc, query asc) order, greedy NMS
    (pipeline.py:266-294).  Returns tuples (class_id, query, box, score, presence)."""
    out = []
    for c in range(score_logits.shape[0]):
        pres = float(sigmoid(presence_logits[c]))
        if pres < presence_thr:
            continue
        s = sigmoid(score_logits[c])
        cands = [(tuple(float(v) for v in boxes[c, q]), float(s[q]), q)
                 for q in range(s.shape[0]) if float(s[q]) >= score_thr]
        cands.sort(key=lambda t: (-t[1], t[2]))
        for box, score, q in greedy_nms(cands, nms_thr):
            out.append((c, q, box, score, pres))
    if cross_class:
        order = sorted(range(len(out)), key=lambda i: (-out[i][3], i))
        kept = greedy_nms([(out[i][2], out[i][3], i) for i in order], nms_thr)
        out = [out[i] for i in sorted(k[2] for k in kept)]
    return out


# ----------------------------------------------------------------------------
# synthetic scenes (scenes.py:15-72)
# ----------------------------------------------------------------------------

PALETTE = np.array([[0.85, 0.15, 0.15], [0.15, 0.35, 0.85], [0.90, 0.60, 0.10], [0.15, 0.75, 0.25],
                    [0.60, 0.20, 0.75], [0.10, 0.75, 0.80], [0.80, 0.75, 0.15], [0.55, 0.35, 0.20]])


def scene(seed: int, image_size: int = 64, num_rects: int = 3, noise: float = 0.05, num_classes: int = 2):
    """Noisy 0.45 background plus painted rectangles, Philox(key=seed) (scenes.py:42-64)."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    s = image_size
    img = 0.45 + noise * rng.uniform(-1.0, 1.0, size=(s, s, 3))
    truth = []
    for _ in range(num_rects):
        cid = int(rng.integers(0, max(num_classes, 1)))
        w, h = float(rng.uniform(0.15, 0.45)), float(rng.uniform(0.15, 0.45))
        cx, cy = float(rng.uniform(w / 2, 1.0 - w / 2)), float(rng.uniform(h / 2, 1.0 - h / 2))
        x0 = int((cx - w / 2) * s)
        y0 = int((cy - h / 2) * s)
        x1 = max(int((cx + w / 2) * s), x0 + 1)
        y1 = max(int((cy + h / 2) * s), y0 + 1)
        img[y0:y1, x0:x1] = PALETTE[cid % len(PALETTE)]
        truth.append({"class_id": cid, "box": (cx, cy, w, h)})
    return np.clip(img, 0.0, 1.0).astype(np.float32).astype(np.float64), truth


def run_detect(P, cfg: OracleConfig, image, names, **thr):
    """Backbone once, all classes, post-process: the `run_batched` composition
    (pipeline.py:202-223)."""
    l0, _, _ = backbone(P, cfg, image)
    texts = [text_embedding(P, cfg, n) for n in names]
    qf, boxes, pres, scores = encdec(P, cfg, l0, texts)
    return postprocess(boxes, scores, pres, **thr)
