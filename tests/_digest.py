"""Digests shared with tests/golden/make_golden.py (same canonical strings)."""
import hashlib

from paper_1303_3182_b200.taskgraph import QR_KINDS

ARITY = (2, 3, 3, 3, 4, 4)


def trace_digest_arrays(kind, idx):
    h = hashlib.sha256()
    for kd, row in zip(kind.tolist(), idx.tolist()):
        h.update(f"{QR_KINDS[kd]}:{','.join(str(x) for x in row[:ARITY[kd]])};".encode())
    return h.hexdigest()


def build_digest(b):
    kind, idx, _ = b.trace_arrays()
    return trace_digest_arrays(kind, idx)


def elim_flat(elim):
    out = []
    for e in elim:
        out += [e.i, e.piv, e.k, e.step]
    return out


def zeroed_flat(b):
    return [[i, k, v] for (i, k), v in sorted(b.zeroed.items())]


def elim_sha(elim):
    h = hashlib.sha256()
    for e in elim:
        h.update(f"{e.k},{e.i},{e.piv},{e.step};".encode())
    return h.hexdigest()


def zeroed_sha(b):
    h = hashlib.sha256()
    for (i, k), v in sorted(b.zeroed.items()):
        h.update(f"{i},{k},{v};".encode())
    return h.hexdigest()
