"""Host-side sequence layer: the input boundary of the hot path.

Same public names and semantics as the reference's ``saix.sequence``
(sequence.py:22-187): ``DnaSequence``, ``RankedText`` (ranks 1..sigma, 0 is
the padding sentinel), ``NPolicy``, ``SequenceError``, ``encode`` / ``decode``
(A1 C2 G3 T4, N5 under KEEP), the seeded ``gen_random`` generator and FASTA
I/O.  These run on the host because they produce the reference's host types;
the device pipeline (``longest_overlap``) encodes ASCII on the GPU instead
(``saix_encode_gsa``).
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from enum import Enum
from typing import IO, Iterable

import numpy as np

ALPHABET = "ACGT"
ALPHABET_N = "ACGTN"


class NPolicy(Enum):
    """Treatment of the ambiguity base N (sequence.py:22-26)."""

    REJECT = "reject"
    KEEP = "keep"


class SequenceError(ValueError):
    """Malformed FASTA or a residue outside the active alphabet."""


@dataclass(frozen=True)
class DnaSequence:
    id: str
    residues: str
    description: str = ""

    def __len__(self) -> int:
        return len(self.residues)


@dataclass(frozen=True, eq=False)
class RankedText:
    """Integer text: ranks 1..sigma, read-only int64 (sequence.py:43-70)."""

    ranks: np.ndarray
    sigma: int
    n: int = field(default=-1)
    _dev: object = field(default=None, repr=False, compare=False)  # resident DeviceText, if any

    def __post_init__(self):
        r = np.asarray(self.ranks, dtype=np.int64)
        r.flags.writeable = False
        object.__setattr__(self, "ranks", r)
        if self.n < 0:
            object.__setattr__(self, "n", int(r.shape[0]))
        if r.shape[0] and (int(r.min()) < 1 or int(r.max()) > self.sigma):
            raise ValueError("ranks must lie in 1..sigma")

    @classmethod
    def _checked(cls, ranks: np.ndarray, sigma: int) -> "RankedText":
        """Construct from int64 ranks already range-checked (on the device)."""
        self = cls.__new__(cls)
        r = np.asarray(ranks, dtype=np.int64)
        r.flags.writeable = False
        object.__setattr__(self, "ranks", r)
        object.__setattr__(self, "sigma", int(sigma))
        object.__setattr__(self, "n", int(r.shape[0]))
        object.__setattr__(self, "_dev", None)
        return self

    def __len__(self) -> int:
        return self.n

    def __eq__(self, other) -> bool:
        if not isinstance(other, RankedText):
            return NotImplemented
        return self.sigma == other.sigma and np.array_equal(self.ranks, other.ranks)


def alphabet(policy: NPolicy) -> str:
    return ALPHABET_N if policy is NPolicy.KEEP else ALPHABET


def _lut(policy: NPolicy) -> np.ndarray:
    lut = np.zeros(256, dtype=np.int64)
    for r, ch in enumerate(alphabet(policy), start=1):
        lut[ord(ch)] = r
    return lut


def encode(seq: DnaSequence, policy: NPolicy = NPolicy.REJECT) -> RankedText:
    """Residues -> ranks A=1 C=2 G=3 T=4 (N=5 under KEEP) (sequence.py:144-157)."""
    raw = np.frombuffer(seq.residues.encode("ascii"), dtype=np.uint8)
    ranks = _lut(policy)[raw]
    if ranks.shape[0]:
        bad = np.flatnonzero(ranks == 0)
        if bad.shape[0]:
            pos = int(bad[0])
            raise SequenceError(
                f"record {seq.id!r}: residue {seq.residues[pos]!r} at position "
                f"{pos} not allowed under policy={policy.value}")
    return RankedText(ranks=ranks, sigma=len(alphabet(policy)))


def residue_error(seq: DnaSequence, pos: int, policy: NPolicy) -> SequenceError:
    """The SequenceError encode() raises for residue `pos` of `seq`."""
    return SequenceError(
        f"record {seq.id!r}: residue {seq.residues[pos]!r} at position "
        f"{pos} not allowed under policy={policy.value}")


def decode(text: RankedText) -> str:
    """Ranks back to letters (sequence.py:160-164)."""
    if text.n == 0:
        return ""
    return np.frombuffer(ALPHABET_N.encode(), np.uint8)[text.ranks - 1].tobytes().decode()


def gen_random(n: int, seed: int,
               weights: tuple[float, float, float, float] = (0.25, 0.25, 0.25, 0.25),
               seq_id: str | None = None) -> DnaSequence:
    """Seeded PCG64 sequence, identical to the reference generator
    (sequence.py:167-187: ``default_rng(seed).choice(4, n, p=w/sum(w))``)."""
    if n < 0:
        raise ValueError("n must be >= 0")
    w = np.asarray(weights, dtype=np.float64)
    if w.shape != (4,) or (w < 0).any() or w.sum() <= 0:
        raise ValueError("weights must be 4 nonnegative values with a positive sum")
    draws = np.random.default_rng(seed).choice(4, size=n, p=w / w.sum())
    letters = np.frombuffer(ALPHABET.encode(), dtype=np.uint8)[draws]
    return DnaSequence(id=seq_id or f"random-{n}-{seed}",
                       residues=letters.tobytes().decode("ascii"),
                       description=f"generated n={n} seed={seed}")


def parse_fasta(source: str | IO[str] | Iterable[str],
                policy: NPolicy = NPolicy.REJECT) -> list[DnaSequence]:
    """FASTA -> records with residue validation (sequence.py:77-125).

    An ASCII ``str`` source is parsed on the device (``fasta.ingest_fasta``:
    line split, strip, classify, upper-case, validate, concatenate); text
    streams and line iterables keep the reference's line-by-line loop here
    (their universal-newline line splitting is the stream's own)."""
    if isinstance(source, str) and source.isascii():
        from .fasta import ingest_fasta
        return ingest_fasta(source, policy, as_ranks=False).records()
    lines = io.StringIO(source) if isinstance(source, str) else source
    ok = set(alphabet(policy))
    out: list[DnaSequence] = []
    rid: str | None = None
    desc = ""
    parts: list[str] = []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line:
            continue
        if line[0] == ">":
            if rid is not None:
                out.append(DnaSequence(rid, "".join(parts), desc))
            head = line[1:].strip()
            if not head:
                raise SequenceError(f"line {lineno}: empty FASTA header")
            rid, _, desc = head.partition(" ")
            desc = desc.strip()
            parts = []
            continue
        if rid is None:
            raise SequenceError(f"line {lineno}: sequence data before any '>' header")
        chunk = line.upper()
        for col, ch in enumerate(chunk, start=1):
            if ch not in ok:
                raise SequenceError(f"record {rid!r}, line {lineno}: "
                                    f"illegal residue {ch!r} at column {col}")
        parts.append(chunk)
    if rid is not None:
        out.append(DnaSequence(rid, "".join(parts), desc))
    return out


def write_fasta(records: Iterable[DnaSequence], width: int = 60) -> str:
    """Records -> FASTA text, inverse of parse_fasta (sequence.py:128-141)."""
    lines: list[str] = []
    for rec in records:
        lines.append(f">{rec.id} {rec.description}" if rec.description else f">{rec.id}")
        s = rec.residues
        lines.extend(s[i:i + width] for i in range(0, len(s), width))
    return "\n".join(lines) + "\n" if lines else ""
