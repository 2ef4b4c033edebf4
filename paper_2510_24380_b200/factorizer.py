"""K8: the factorizer's hierarchy encoding on the B200.

Mirror of the reference's ``factorizer.encode_hierarchy(factorizer, library)``
(reference ``pkg/src/apexcsl/factorizer.py:218-233``, forward pass
``Factorizer.forward_cache`` :157-171, networks ``nn.MLP`` nn.py:44-62,
features ``props.library_synthon_features`` props.py:43-67), computed by
``apex_encode_hierarchy`` (csrc/k8.cuh): synthon feature hashing (BLAKE2b on
the device), the synthon MLP, the R-group and reaction deep sets, the value
and key MLPs and the pair rows ``u = v[member] @ K_r^T``, in fp64.

``encode_hierarchy`` returns a ``HierarchyCache`` of the caller's class (host
copies, like the reference).  ``precompute_from_factorizer`` chains K8 and K1
with the pair matrix resident on the device (no host round trip of ``u``:
680 MB at the 5e9-product shape) and returns the contribution table.

The factorizer may be the reference's object or anything with the same
attributes (``synthon_encoder``, ``rgroup_encoder.phi/.rho``,
``reaction_encoder.phi/.rho``, ``value_encoder``, ``key_encoder`` each with
``dims`` and ``params`` [W0, b0, ...] or [W0, W1, ...] without bias,
``dims.d`` / ``dims.d_u``, ``feature_config.p`` / ``.seed``).
"""

from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np

from . import _native
from .csl import library_fingerprint
from .engine import _error, default_device

FEATURE_SCALE = 0.25  # props._FEATURE_SCALE (props.py:24)


@dataclass
class HierarchyCache:
    h_s: np.ndarray
    h_r: np.ndarray
    h_t: np.ndarray
    u: np.ndarray
    member_ids: np.ndarray
    rg_offsets: np.ndarray
    rg_pos: dict
    fingerprint: str
    synthon_encoder_evals: int


def _networks(f):
    return [f.synthon_encoder, f.rgroup_encoder.phi, f.rgroup_encoder.rho, f.reaction_encoder.phi,
            f.reaction_encoder.rho, f.value_encoder, f.key_encoder]


def _flat_params(nets):
    """[W0, b0, W1, b1, ...] of every network, biases zero-filled for bias-free MLPs."""
    shapes, flat = [], []
    for mlp in nets:
        dims = list(mlp.dims)
        shapes.append(dims)
        params = list(mlp.params)
        with_bias = len(params) == 2 * (len(dims) - 1)
        for i in range(len(dims) - 1):
            W = np.asarray(params[2 * i] if with_bias else params[i], dtype=np.float64)
            b = np.asarray(params[2 * i + 1], dtype=np.float64) if with_bias else np.zeros(dims[i + 1])
            flat.append(W.reshape(-1))
            flat.append(b.reshape(-1))
    return shapes, np.concatenate(flat)


def _context(library):
    """factorizer.build_context without the host feature hashing (done on the
    device): pair-row layout, R-group / reaction offsets, token bytes."""
    member_ids, rg_offsets, rg_parent, rx_offsets, rg_pos = [], [0], [], [0], {}
    for ti, rx in enumerate(library.reactions):
        for rg in rx.rgroups:
            rg_pos[rg.rgroup_id] = len(rg_parent)
            member_ids.extend(rg.synthon_ids)
            rg_offsets.append(len(member_ids))
            rg_parent.append(ti)
        rx_offsets.append(len(rg_parent))
    toks = [s.token.encode() for s in library.synthons]
    ids = [s.synthon_id for s in library.synthons]
    if ids != list(range(len(ids))):
        raise _error("synthon ids must be dense 0..|S|-1 (feature rows are indexed by id)")
    if any(len(t) > 64 for t in toks):
        raise _error("synthon token longer than 64 bytes")
    off = np.zeros(len(toks) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(t) for t in toks])
    return (np.asarray(member_ids, dtype=np.int64), np.asarray(rg_offsets, dtype=np.int64),
            np.asarray(rg_parent, dtype=np.int32), np.asarray(rx_offsets, dtype=np.int64), rg_pos,
            np.frombuffer(b"".join(toks), dtype=np.uint8), off)


def _run(factorizer, library, device, want):
    member_ids, rg_offsets, rg_parent, rx_offsets, rg_pos, tb, toff = _context(library)
    shapes, params = _flat_params(_networks(factorizer))
    fc = factorizer.feature_config
    dev = default_device() if device is None else device
    ctx = _native.DeviceContext(int(dev[0] if isinstance(dev, (list, tuple)) else dev))
    try:
        out = ctx.encode_hierarchy(shapes, params, tb, toff, f"{fc.seed}:".encode(), fc.p, FEATURE_SCALE, member_ids,
                                   rg_offsets, rg_parent, rx_offsets, factorizer.dims.d, factorizer.dims.d_u, want)
    except _native.NativeError as exc:
        ctx.close()
        raise _error(str(exc)) from None
    return ctx, out, member_ids, rg_offsets, rg_pos


def encode_hierarchy(factorizer, library, device=None):
    """The factorizer's full-hierarchy forward pass on the device
    (factorizer.py:218-233); returns a HierarchyCache of the caller's class."""
    ctx, out, member_ids, rg_offsets, rg_pos = _run(factorizer, library, device, ("u", "h_s", "h_r", "h_t"))
    ctx.close()
    mod = sys.modules.get(type(factorizer).__module__)
    cls = getattr(mod, "HierarchyCache", HierarchyCache) if mod else HierarchyCache
    return cls(h_s=out["h_s"], h_r=out["h_r"], h_t=out["h_t"], u=out["u"], member_ids=member_ids,
               rg_offsets=rg_offsets, rg_pos=rg_pos, fingerprint=library_fingerprint(library),
               synthon_encoder_evals=len(library.synthons))


def precompute_from_factorizer(factorizer, surrogate, library, device=None):
    """K8 then K1 on the device with the pair matrix resident: the reference's
    encode_hierarchy + precompute_contributions (engine.py:80-92) without a
    host copy of u.  Returns a ContributionTable of the caller's class."""
    from . import engine

    ctx, _, member_ids, rg_offsets, rg_pos = _run(factorizer, library, device, ())
    try:
        values = ctx.precompute_resident(np.asarray(surrogate.head_w, dtype=np.float64),
                                         np.asarray(surrogate.head_b, dtype=np.float64))
    except _native.NativeError as exc:
        raise _error(str(exc)) from None
    finally:
        ctx.close()
    rg_ids = np.asarray(sorted(rg_pos, key=rg_pos.get))
    mod = sys.modules.get(type(surrogate).__module__.replace("surrogate", "engine"))
    cls = getattr(mod, "ContributionTable", engine.ContributionTable) if mod else engine.ContributionTable
    return cls(values=values, biases=np.asarray(surrogate.head_b, dtype=np.float64).copy(),
               task_names=list(surrogate.task_names), member_ids=member_ids, rg_offsets=rg_offsets, rg_ids=rg_ids,
               fingerprint=library_fingerprint(library))
