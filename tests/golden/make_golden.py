"""Generate tests/golden/golden.npz from the UNMODIFIED reference library.

Run here (the container that has /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Every array in golden.npz is produced by oracle/_ref/liblane_ref.so, i.e. the
reference's own sources (proj/src/*.cpp) compiled with its Release flags and
driven through its public API (ref_shim.cpp).  The fixture pins the C
restatement (oracle/lane_oracle.c) on machines where /root/reference is absent
(the GPU box): tests/test_oracle.py checks the restatement against it
bit-for-bit.  Known-answer values from the reference's own tests are included
verbatim where they exist (cited inline).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402

IRIS = os.path.join(HERE, "iris_normalized.txt")


def rng_u64(seed, n):
    out = np.zeros(n, np.uint64)
    po.ref_lib().lr_rng_u64(seed, n, out)
    return out


def rng_fill(seed, n, lo, hi):
    out = np.zeros(n, np.float32)
    po.ref_lib().lr_rng_fill(seed, n, lo, hi, out)
    return out


def main():
    g = {}
    # --- SplitMix64 / random_fill (test_tensor.cpp:115-141) ---------------
    for s in (42, 7, 0, 2026):
        g[f"rng_u64_{s}"] = rng_u64(s, 16)
        g[f"rng_fill_{s}"] = rng_fill(s, 16, -0.5, 0.5)
    g["rng_fill_42_unit"] = rng_fill(42, 4, 0.0, 1.0)  # == test_tensor.cpp:121-124

    # --- layer backward: random acceptance-style cases (acceptance.cpp:250-304)
    rs = np.random.default_rng(1234)
    for c in range(24):
        I, O = int(rs.integers(1, 33)), int(rs.integers(2, 33))
        outputs = rs.uniform(0, 1, O).astype(np.float32)
        inputs = rs.uniform(-1, 1, I).astype(np.float32)
        target = np.zeros(O, np.float32)
        target[rs.integers(0, O)] = 1
        r = po.ref_layer_backward("softmax", outputs, inputs, 0.05, target=target)
        g[f"smb{c}_in"] = np.concatenate([outputs, inputs, target])
        g[f"smb{c}_shape"] = np.array([I, O])
        for k, v in r.items():
            g[f"smb{c}_{k}"] = v
    for c in range(24):
        I, O, N = int(rs.integers(1, 33)), int(rs.integers(1, 33)), int(rs.integers(1, 9))
        outputs = rs.uniform(-0.99, 0.99, O).astype(np.float32)
        inputs = rs.uniform(-1, 1, I).astype(np.float32)
        nW = rs.uniform(-1, 1, (O, N)).astype(np.float32)
        nd = rs.uniform(-1, 1, N).astype(np.float32)
        r = po.ref_layer_backward("fc", outputs, inputs, 0.05, next_W=nW, next_d=nd)
        g[f"fcb{c}_in"] = np.concatenate([outputs, inputs, nW.reshape(-1), nd])
        g[f"fcb{c}_shape"] = np.array([I, O, N])
        for k, v in r.items():
            g[f"fcb{c}_{k}"] = v

    # --- layer forward (layers.cpp:27-87): bitwise through glibc tanhf/expf
    for c in range(16):
        I, O = int(rs.integers(1, 65)), int(rs.integers(2, 65))
        W = rs.uniform(-2, 2, (I, O)).astype(np.float32)
        b = rs.uniform(-1, 1, O).astype(np.float32)
        x = rs.uniform(-1, 1, I).astype(np.float32)
        kind = "softmax" if c % 2 else "fc"
        z, a = po.ref_layer_forward(kind, W, b, x)
        g[f"fwd{c}_W"], g[f"fwd{c}_b"], g[f"fwd{c}_x"] = W, b, x
        g[f"fwd{c}_z"], g[f"fwd{c}_a"] = z, a

    # --- network steps at the BASELINE shapes (seed 42, synthetic seed 9) ---
    for name, (F, H, Cc, eta, steps) in {
        "c1": (4, [8], 3, 0.01, 4),
        "c2": (784, [128], 10, 0.01, 3),
        "c4": (340, [256], 10, 1e-4, 2),
        "deep": (16, [12, 9], 5, 0.05, 4),
    }.items():
        X, T = po.synthetic_dataset(F, Cc, 8, 9)
        net = po.RefNet(F, H, Cc, seed=42)
        g[f"{name}_hash0"] = np.array([net.hash()], np.uint64)
        hashes, probs, deltas = [], [], []
        for s in range(steps):
            probs.append(net.forward(X[s]))
            net.backward_plan_run(T[s], eta)
            hashes.append(net.hash())
            deltas.append(np.concatenate([net.get(l, po.DELTAS) for l in range(len(H) + 1)]))
        g[f"{name}_hashes"] = np.array(hashes, np.uint64)
        g[f"{name}_probs"] = np.stack(probs)
        g[f"{name}_deltas"] = np.stack(deltas)

    # --- C1: Iris 4-8-3, one epoch of SGD (BASELINE configs[0]) -----------
    X, T = po.load_dataset(IRIS, 4, 3)
    Xtr, Ttr, Xte, Tte = po.split(X, T, 0.9, 42)
    net = po.RefNet(4, [8], 3, seed=42)
    st = net.train(Xtr, Ttr, 0.1, max_epochs=1, seed=42)
    g["iris1_stats"] = np.array(st[0][1:], np.float32)
    g["iris1_W0"], g["iris1_W1"] = net.get(0, po.W), net.get(1, po.W)
    g["iris1_b0"], g["iris1_b1"] = net.get(0, po.B), net.get(1, po.B)
    g["iris1_hash"] = np.array([net.hash()], np.uint64)
    # acceptance C5 (acceptance.cpp:443-469): eta 0.1, max_error 0.05, 2000 epochs
    net = po.RefNet(4, [8], 3, seed=42)
    st = net.train(Xtr, Ttr, 0.1, max_epochs=2000, max_error=0.05, seed=42)
    g["irisC5_epochs"] = np.array([len(st)])
    g["irisC5_curve"] = np.array([s[1] for s in st], np.float32)
    g["irisC5_test"] = np.array(net.evaluate(Xte, Tte), np.float32)

    # --- XOR regression oracle (test_training.cpp:204-221): seed 111 -> 77 --
    Xx = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.float32)
    Tx = np.array([[1, 0], [0, 1], [0, 1], [1, 0]], np.float32)
    net = po.RefNet(2, [4], 2, seed=111)
    st = net.train(Xx, Tx, 0.5, max_epochs=5000, max_error=0.05, seed=111)
    g["xor_epochs"] = np.array([len(st)])
    g["xor_curve"] = np.array([s[1] for s in st], np.float32)
    g["xor_eval"] = np.array(net.evaluate(Xx, Tx), np.float32)

    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes; "
          f"xor epochs {g['xor_epochs'][0]}, iris C5 epochs {g['irisC5_epochs'][0]} "
          f"test acc {g['irisC5_test'][1]:.3f}")


if __name__ == "__main__":
    main()
