"""CPU oracle for the Sample-Align-D k-mer-rank domain decomposition (ctypes wrapper).

TEST INFRASTRUCTURE ONLY. Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this package.
The product (``paper_0901_2742_b200``) never imports it.

The arithmetic lives in ``sad_oracle.c`` (plain C, see its header for the
paper citations); this file only compiles it with gcc and marshals numpy
arrays.  Parity status: every function is pinned (tests/test_oracle_*.py):
hand values, the worked example, closed forms, invariants and a Python
brute force on small inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sad_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

ALPHABETS = {"protein": 0, "dna": 1}
ERRORS = {-1: "ARG", -3: "SYMBOL", -4: "TOO_SHORT", -5: "TOO_LONG", -6: "INSUFFICIENT", -7: "EMPTY", -11: "OOM"}

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_POSIX_C_SOURCE=200809L", "-fopenmp",
                               "-shared", "-fPIC", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.or_abi.restype = i32
        L.or_q.restype = ctypes.c_uint64
        L.or_q.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.or_count.restype = i64
        L.or_count.argtypes = [P, i64, i32, P, P]
        L.or_pair.restype = i32
        L.or_pair.argtypes = [P, i64, P, i64, i32, P, P]
        L.or_run.restype = i32
        L.or_run.argtypes = [P, P, i64, i32, i32, i32, i32] + [P] * 14
        L.or_run2.restype = i32
        L.or_run2.argtypes = [P, P, i64, i32, i32, i32, i32, i32] + [P] * 15
        L.or_rows_T.restype = i32
        L.or_rows_T.argtypes = [P, P, i64, i32, i32, P, i64, i32, P]
        L.or_rank_vs_set.restype = i32
        L.or_rank_vs_set.argtypes = [P, P, i64, i32, P, i64, i32, P]
        L.or_pairs_S.restype = i32
        L.or_pairs_S.argtypes = [P, P, i32, P, P, i64, i32, P, P]
        L.or_rank_R.restype = ctypes.c_double
        L.or_rank_R.argtypes = [ctypes.c_double]
        L.or_threads.restype = i32
        L.or_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _b(s):
    if isinstance(s, str):
        s = s.encode()
    return np.frombuffer(bytes(s), dtype=np.uint8).copy() if len(s) else np.zeros(1, np.uint8)


class OracleError(RuntimeError):
    def __init__(self, code, idx=-1, pos=-1):
        super().__init__(f"oracle error {ERRORS.get(code, code)} (seq {idx}, pos {pos})")
        self.code, self.name, self.idx, self.pos = code, ERRORS.get(code, str(code)), idx, pos


def q(S: int, den: int) -> int:
    """floor(2^32 * S / den) — SURVEY reading A5."""
    return int(lib().or_q(S, den))


def count(x, k: int) -> dict:
    """k-mer multiset of one sequence as {kmer string: count}."""
    xb = _b(x)
    L = len(x)
    n = max(L - k + 1, 1)
    pos = np.zeros(n, np.int64)
    cnt = np.zeros(n, np.int64)
    d = lib().or_count(_p(xb), L, k, _p(pos), _p(cnt))
    if d < 0:
        raise OracleError(int(d))
    s = bytes(xb[:L])
    return {s[pos[i]: pos[i] + k].decode(): int(cnt[i]) for i in range(d)}


def pair(x, y, k: int):
    """(S, den) of one pair — PAPER.md:42."""
    xb, yb = _b(x), _b(y)
    S = np.zeros(1, np.int64)
    d = np.zeros(1, np.int64)
    rc = lib().or_pair(_p(xb), len(x), _p(yb), len(y), k, _p(S), _p(d))
    if rc:
        raise OracleError(rc)
    return int(S[0]), int(d[0])


@dataclass
class Result:
    T: np.ndarray
    anc: np.ndarray
    ga: int
    S: np.ndarray
    den: np.ndarray
    sorted: np.ndarray
    samples: np.ndarray
    pivots: np.ndarray
    bucket: np.ndarray
    border: np.ndarray
    bsize: np.ndarray
    stage_ms: np.ndarray
    rsamples: np.ndarray | None = None

    def buckets(self):
        out, o = [], 0
        for b in self.bsize:
            out.append(self.border[o: o + int(b)].tolist())
            o += int(b)
        return out


def run(ascii_, offsets, alphabet: str, k: int, p: int, nthreads: int = 0, mode: str = "ga") -> Result:
    """The whole oracle pipeline on one process. mode "ga": rank against
    the global ancestor (readings A7, A8); "samples": the paper's literal rank against the k*p
    gathered samples (reading A27; S and den then hold (T', 1), T' the exact
    fixed-point sum of q over the samples)."""
    a = np.ascontiguousarray(ascii_, dtype=np.uint8)
    if a.size == 0:
        a = np.zeros(1, np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    n = len(o) - 1
    z = lambda m, t=np.int64: np.zeros(max(m, 1), t)
    T, anc, ga, Sg, dg = z(n, np.uint64), z(p), z(1), z(n), z(n)
    srt, smp, piv, bk, bo, bs = z(n), z(p * (p - 1)), z(p - 1), z(n), z(n), z(p)
    ms = np.zeros(4, np.float64)
    ei, ep = np.full(1, -1, np.int64), np.full(1, -1, np.int64)
    rs = z(p * (p - 1))
    rc = lib().or_run2(_p(a), _p(o), n, ALPHABETS[alphabet], k, p, {"ga": 0, "samples": 1}[mode], nthreads,
                       _p(T), _p(anc), _p(ga), _p(Sg), _p(dg), _p(srt), _p(smp), _p(piv), _p(bk), _p(bo), _p(bs),
                       _p(rs), _p(ms), _p(ei), _p(ep))
    if rc:
        raise OracleError(rc, int(ei[0]), int(ep[0]))
    return Result(T[:n], anc[:p], int(ga[0]), Sg[:n], dg[:n], srt[:n], smp[: p * (p - 1)], piv[: p - 1],
                  bk[:n], bo[:n], bs[:p], ms, rs[: p * (p - 1)] if mode == "samples" else None)


def rows_T(ascii_, offsets, k: int, p: int, rows, nthreads: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(ascii_, dtype=np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(max(len(r), 1), np.uint64)
    rc = lib().or_rows_T(_p(a), _p(o), len(o) - 1, k, p, _p(r), len(r), nthreads, _p(out))
    if rc:
        raise OracleError(rc)
    return out[: len(r)]


def rank_vs_set(ascii_, offsets, k: int, ref, nthreads: int = 0) -> np.ndarray:
    """T'_i = sum over the reference set `ref` (source indices) of q(x_i, s), for every sequence."""
    a = np.ascontiguousarray(ascii_, dtype=np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    r = np.ascontiguousarray(ref, dtype=np.int64)
    n = len(o) - 1
    out = np.zeros(max(n, 1), np.uint64)
    rc = lib().or_rank_vs_set(_p(a), _p(o), n, k, _p(r), len(r), nthreads, _p(out))
    if rc:
        raise OracleError(rc)
    return out[:n]


def pairs_S(ascii_, offsets, k: int, pi, pj, nthreads: int = 0):
    a = np.ascontiguousarray(ascii_, dtype=np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    pi = np.ascontiguousarray(pi, dtype=np.int64)
    pj = np.ascontiguousarray(pj, dtype=np.int64)
    S = np.zeros(max(len(pi), 1), np.int64)
    d = np.zeros(max(len(pi), 1), np.int64)
    rc = lib().or_pairs_S(_p(a), _p(o), k, _p(pi), _p(pj), len(pi), nthreads, _p(S), _p(d))
    if rc:
        raise OracleError(rc)
    return S[: len(pi)], d[: len(pi)]


def rank_R(D: float) -> float:
    return float(lib().or_rank_R(D))


def threads(nthreads: int = 0) -> int:
    return int(lib().or_threads(nthreads))
