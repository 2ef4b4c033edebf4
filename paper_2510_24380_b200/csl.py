"""Host-side index space of a combinatorial synthesis library (CSL).

A mirror of the reference data model (`apexcsl/csl.py`) restricted to what the
retrieval path needs, so the B200 path runs where the reference package is not
installed (the GPU box).  Objects of the reference classes are accepted
everywhere by duck typing (same attribute names).

Index space (csl.py:1-8, 151-184): reactions in declaration order; inside a
reaction a mixed-radix number whose most significant digit is the first
R-group.  ``g = reaction_offset(t) + mixed_radix(digits)``.
"""

from __future__ import annotations

import hashlib
import weakref
from dataclasses import dataclass, field

import numpy as np

MAX_COUNT = 2**64 - 1
LIBRARY_FORMAT_VERSION = "cslv1"


class LibraryError(ValueError):
    """Structural problem in a library definition or an index out of range."""


@dataclass(frozen=True)
class SynthonRecord:
    synthon_id: int
    token: str


@dataclass(frozen=True)
class RgroupSpec:
    rgroup_id: int
    synthon_ids: tuple[int, ...]


@dataclass(frozen=True)
class ReactionSpec:
    reaction_id: int
    rgroups: tuple[RgroupSpec, ...]


@dataclass(frozen=True)
class MultiIndex:
    """One product: a reaction plus an (rgroup_id, synthon_id) pair per R-group."""

    reaction_id: int
    assignment: tuple[tuple[int, int], ...]

    def synthon_ids(self) -> tuple[int, ...]:
        return tuple(s for _, s in self.assignment)


@dataclass
class CslLibrary:
    reactions: tuple[ReactionSpec, ...]
    synthons: tuple[SynthonRecord, ...]

    _sizes: tuple[int, ...] = field(init=False, repr=False, compare=False)
    _offsets: tuple[int, ...] = field(init=False, repr=False, compare=False)
    _digit: dict = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        sizes, offsets, digit = [], [0], {}
        for rx in self.reactions:
            n = 1
            for rg in rx.rgroups:
                n *= len(rg.synthon_ids)
                digit[rg.rgroup_id] = {s: i for i, s in enumerate(rg.synthon_ids)}
            sizes.append(n)
            offsets.append(offsets[-1] + n)
        self._sizes = tuple(sizes)
        self._offsets = tuple(offsets)
        self._digit = digit

    def reaction(self, reaction_id: int) -> ReactionSpec:
        return self.reactions[reaction_id]

    def reaction_size(self, reaction_id: int) -> int:
        return self._sizes[reaction_id]

    def reaction_offset(self, reaction_id: int) -> int:
        return self._offsets[reaction_id]

    def synthon_digit(self, rgroup_id: int, synthon_id: int) -> int:
        try:
            return self._digit[rgroup_id][synthon_id]
        except KeyError:
            raise LibraryError(f"synthon {synthon_id} is not eligible for R-group {rgroup_id}") from None

    def iter_rgroups(self):
        for rx in self.reactions:
            yield from rx.rgroups


def product_count(library) -> int:
    """Sum over reactions of the product of R-group sizes (csl.py:138-148)."""
    total = 0
    for rx in library.reactions:
        n = 1
        for rg in rx.rgroups:
            n *= len(rg.synthon_ids)
        total += n
    if total > MAX_COUNT:
        raise LibraryError(f"product count {total} exceeds unsigned 64-bit range")
    return total


def reaction_offsets(library) -> list[int]:
    out = [0]
    for rx in library.reactions:
        n = 1
        for rg in rx.rgroups:
            n *= len(rg.synthon_ids)
        out.append(out[-1] + n)
    return out


def decode_index(library, gidx: int) -> MultiIndex:
    """g -> MultiIndex (inverse of the mixed-radix codec, csl.py:166-184)."""
    offs = reaction_offsets(library)
    if not 0 <= gidx < offs[-1]:
        raise LibraryError(f"global index {gidx} out of range [0, {offs[-1]})")
    t = int(np.searchsorted(np.asarray(offs, dtype=object), gidx, side="right")) - 1
    rx = library.reactions[t]
    rem = gidx - offs[t]
    digits = [0] * len(rx.rgroups)
    for j in range(len(rx.rgroups) - 1, -1, -1):
        rem, digits[j] = divmod(rem, len(rx.rgroups[j].synthon_ids))
    return MultiIndex(rx.reaction_id, tuple((rg.rgroup_id, rg.synthon_ids[d]) for rg, d in zip(rx.rgroups, digits)))


def serialize_library(library) -> str:
    """Canonical text (the `cslv1` line format); its SHA-256 is the fingerprint."""
    n_rg = sum(len(rx.rgroups) for rx in library.reactions)
    out = [f"{LIBRARY_FORMAT_VERSION} {len(library.synthons)} {n_rg} {len(library.reactions)}"]
    out.extend(f"S {s.synthon_id} {s.token}" for s in library.synthons)
    for rx in library.reactions:
        for rg in rx.rgroups:
            out.append(" ".join(["R", str(rg.rgroup_id), *map(str, rg.synthon_ids)]))
    for rx in library.reactions:
        out.append(" ".join(["T", str(rx.reaction_id), *(str(rg.rgroup_id) for rg in rx.rgroups)]))
    return "\n".join(out) + "\n"


def deserialize_library(text: str) -> CslLibrary:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise LibraryError("empty library file")
    head = lines[0].split()
    if len(head) != 4 or head[0] != LIBRARY_FORMAT_VERSION:
        raise LibraryError(f"bad header: {lines[0]!r}")
    synthons, rgroups, reactions = [], {}, []
    for ln in lines[1:]:
        kind, *rest = ln.split()
        if kind == "S":
            synthons.append(SynthonRecord(int(rest[0]), rest[1]))
        elif kind == "R":
            rgroups[int(rest[0])] = RgroupSpec(int(rest[0]), tuple(map(int, rest[1:])))
        elif kind == "T":
            reactions.append(ReactionSpec(int(rest[0]), tuple(rgroups[int(r)] for r in rest[1:])))
        else:
            raise LibraryError(f"unknown record type {kind!r}")
    return CslLibrary(tuple(reactions), tuple(synthons))


_FP_CACHE: dict[int, tuple[weakref.ref, str]] = {}


def library_fingerprint(library, memo: bool = True) -> str:
    """SHA-256 of the canonical serialization (csl.py:380-382).

    The reference recomputes it on every search call (0.19 s at 1e9 products,
    0.79 s at 5e9); libraries are immutable after construction (SPEC), so it is
    memoized per object here.
    """
    if memo:
        hit = _FP_CACHE.get(id(library))
        if hit is not None and hit[0]() is library:
            return hit[1]
    fp = hashlib.sha256(serialize_library(library).encode()).hexdigest()
    if memo:
        try:
            _FP_CACHE[id(library)] = (weakref.ref(library), fp)
        except TypeError:
            pass
    return fp
