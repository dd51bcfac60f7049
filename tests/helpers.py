"""Shared helpers for the test suite (CPU side)."""
import math

import numpy as np

import paper_2509_04955_b200 as pkg
from oracle import pyoracle

MNEMONIC_1Q = ["h", "x", "y", "z", "s", "sdg", "t", "tdg"]
MNEMONIC_1Q_P = ["rx", "ry", "rz", "u1", "p"]
MNEMONIC_2Q = ["cx", "cz"]
MNEMONIC_2Q_P = ["cp", "cu1"]


def rand_state(n, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return a / np.linalg.norm(a)


def rand_unitary(k, rng):
    d = 1 << k
    q, r = np.linalg.qr(rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d)))
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_mnemonic_circuit(n, ngates, seed):
    """Random circuit over the full QASM mnemonic set (acceptance #1)."""
    rng = np.random.default_rng(seed)
    c = pkg.Circuit.empty(n)
    for _ in range(ngates):
        kind = rng.integers(0, 4) if n >= 2 else rng.integers(0, 2)
        if kind == 0:
            c.add(str(rng.choice(MNEMONIC_1Q)), [int(rng.integers(n))])
        elif kind == 1:
            c.add(str(rng.choice(MNEMONIC_1Q_P)), [int(rng.integers(n))], [float(rng.uniform(0, 2 * math.pi))])
        else:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            if kind == 2:
                c.add(str(rng.choice(MNEMONIC_2Q)), [a, b])
            else:
                c.add(str(rng.choice(MNEMONIC_2Q_P)), [a, b], [float(rng.uniform(0, 2 * math.pi))])
    return c


def random_unitary_circuit(n, ngates, seed, kmax=3, ctrl=True):
    """Random dense k-qubit unitaries (k <= kmax) with optional controls."""
    rng = np.random.default_rng(seed)
    c = pkg.Circuit.empty(n)
    for _ in range(ngates):
        k = int(rng.integers(1, min(kmax, n) + 1))
        nc = int(rng.integers(0, min(2, n - k) + 1)) if ctrl else 0
        qs = [int(x) for x in rng.choice(n, k + nc, replace=False)]
        c.add_unitary(rand_unitary(k, rng), qs[:k], qs[k:])
    return c


def qft_basis_expected(n, x, offset=0, count=None):
    """QFT|x> amplitudes [offset, offset + count) (all of them by default)."""
    count = (1 << n) - offset if count is None else count
    y = np.arange(offset, offset + count, dtype=np.uint64)
    ph = (np.uint64(x) * y) & np.uint64((1 << n) - 1)
    return np.exp(2j * np.pi * ph.astype(np.float64) / (1 << n)) / math.sqrt(1 << n)


def oracle_run(c, amps=None, threads=None):
    return pyoracle.run_local(c, amps, threads)


def unitarity_defect(circ) -> float:
    """sum over gates of max(s_max^2 - 1, 1 - s_min^2) of the gate's fp64 matrix: the norm
    drift that the circuit's own (rounded) gate matrices allow even in exact arithmetic.
    Deep circuits reach ~1e-11 (uccsd:20:100000:3: 9.6e-12; the CPU oracle drifts -7.8e-12
    there), so norm conservation is asserted against 1e-12 + this bound."""
    _, recs, nr, pool = circ.export()
    cache = {}
    total = 0.0
    for i in range(nr):
        r = recs[i]
        if r.arity == 0:
            continue
        d = 1 << r.arity
        key = (r.mat_off, d)
        if key not in cache:
            sv = np.linalg.svd(pool[r.mat_off:r.mat_off + d * d].reshape(d, d), compute_uv=False)
            cache[key] = max(sv.max() ** 2 - 1.0, 1.0 - sv.min() ** 2, 0.0)
        total += cache[key]
    return total
