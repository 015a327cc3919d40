"""Seeded synthetic digit generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no FFT, no intervals, no carry):
it only draws base-256 digit vectors.  Both sides of every parity test take
their inputs from here (the device generator ``ivm_generate_digits`` in the
C ABI implements the same counter-based generator, pinned bit-exact against
this file by ``tests/test_inputs.py``).

Generator, all arithmetic mod 2^64:

    mix64(z): z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
              z *= 0x94D049BB133111EB; z ^= z>>31
    r(seed, s, i) = mix64(seed + 0x9E3779B97F4A7C15 * ((s << 32) + i + 1))
    s = 2*pair + operand (a = 0, b = 1); i = digit index

    uniform : r >> 56
    all255  : 255
    sparse  : (r & 0xFFFFFFFF) < 429496730 ? r >> 56 : 0      (90 % zeros)
    msd     : uniform, and if d[n-1] == 0: d[n-1] = 1 + r(seed, s, n) % 255

The paper's workloads are "uniformly-random n-digit base-256 inputs"
(§3) plus the worst case all-255 and a sparse mix named in
BASELINE.json's configs; no public dataset is involved.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
SPARSE_THRESHOLD = 429496730  # floor(0.1 * 2^32) + 1 -> P(nonzero) ~= 0.1

KINDS = {"uniform": 0, "all255": 1, "sparse": 2, "msd": 3}

SEED_BASE = 0x10060405


def config_seed(k: int) -> int:
    """Seed of config C<k> (seed_Ck = 0x10060405 + k)."""
    return SEED_BASE + k


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * M1
        z = z ^ (z >> np.uint64(27))
        z = z * M2
        z = z ^ (z >> np.uint64(31))
    return z


def rand64(seed: int, s: np.ndarray, i: np.ndarray) -> np.ndarray:
    """r(seed, s, i) for broadcastable arrays s (stream) and i (digit index)."""
    s = np.asarray(s, dtype=np.uint64)
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = (s << np.uint64(32)) + i + np.uint64(1)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + GOLDEN * ctr
    return mix64(z)


def digits(seed: int, pairs: np.ndarray, operand: int, n: int, kind) -> np.ndarray:
    """Digit vectors for the given pair indices: uint8 array [len(pairs), n].

    ``kind`` is a name from KINDS or an int array (one kind per pair).
    """
    pairs = np.asarray(pairs, dtype=np.uint64).reshape(-1)
    B = pairs.shape[0]
    if isinstance(kind, str):
        kinds = np.full(B, KINDS[kind], dtype=np.int64)
    else:
        kinds = np.asarray(kind, dtype=np.int64).reshape(-1)
        assert kinds.shape[0] == B
    s = (np.uint64(2) * pairs + np.uint64(operand))[:, None]
    idx = np.arange(n, dtype=np.uint64)[None, :]
    r = rand64(seed, s, idx)
    uni = (r >> np.uint64(56)).astype(np.uint8)
    out = uni.copy()
    k = kinds[:, None]
    out = np.where(k == KINDS["all255"], np.uint8(255), out)
    low = (r & np.uint64(0xFFFFFFFF))
    sparse = np.where(low < np.uint64(SPARSE_THRESHOLD), uni, np.uint8(0)).astype(np.uint8)
    out = np.where(k == KINDS["sparse"], sparse, out).astype(np.uint8)
    msd_rows = np.nonzero(kinds == KINDS["msd"])[0]
    if msd_rows.size and n > 0:
        top = out[msd_rows, n - 1]
        zero = msd_rows[top == 0]
        if zero.size:
            rr = rand64(seed, s[zero, 0], np.uint64(n))
            out[zero, n - 1] = (np.uint64(1) + rr % np.uint64(255)).astype(np.uint8)
    return out


def pair_digits(seed: int, pairs, n: int, kind):
    """(a, b) digit matrices for the given pairs."""
    return digits(seed, pairs, 0, n, kind), digits(seed, pairs, 1, n, kind)


# --------------------------------------------------------------------------
# Workload configurations (BASELINE.json "configs")
# --------------------------------------------------------------------------

def class_of_pairs(config: str, batch: int) -> np.ndarray:
    """Digit-distribution kind per pair for a named config."""
    p = np.arange(batch)
    if config == "C1":
        return np.full(batch, KINDS["msd"])
    if config == "C2":
        return np.full(batch, KINDS["uniform"])
    if config in ("C3", "C4"):
        return np.where(p < batch // 2, KINDS["uniform"], KINDS["all255"])
    if config == "C5":
        return np.array([KINDS["uniform"], KINDS["all255"], KINDS["sparse"]])[p % 3]
    raise KeyError(config)


CONFIGS = {
    # id: (n list, batch, precision)
    "C1": ([1000], 1, "f64"),
    "C2": ([4096], 4096, "f64"),
    "C3": ([75000], 64, "f64"),
    "C4": ([32, 64, 96, 120, 160, 256], 1024, "f32"),
    "C5": ([16384], 65536, "f64"),
}


def config_inputs(config: str, n: int | None = None, pairs=None):
    """(a, b, kinds) for config C<k> (optionally a subset of pair indices)."""
    ns, batch, _ = CONFIGS[config]
    if n is None:
        n = ns[0]
    k = int(config[1:])
    kinds_all = class_of_pairs(config, batch)
    if pairs is None:
        pairs = np.arange(batch)
    pairs = np.asarray(pairs)
    kinds = kinds_all[pairs]
    a, b = pair_digits(config_seed(k), pairs, n, kinds)
    return a, b, kinds
