"""Diagnostics for the decode GEMV: structured inputs written straight into the packed
buffers (no pack), plain launches, printed comparisons.  Run on the GPU box."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10645_b200 as paro  # noqa: E402


def make_packed(codes_u8, S, z, n_rot=0):
    """codes_u8 [N,K] ints 0..15, S fp16 [N,G], z ints [N,G] -> PackedLinear (no transform)."""
    N, K = codes_u8.shape
    G = K // 128
    pk = paro.alloc_packed(N, K, n_rot)
    c = (codes_u8[:, 0::2] | (codes_u8[:, 1::2] << 4)).astype(np.uint8)
    pk.codes[: N * K // 2].copy_(torch.from_numpy(c.reshape(-1)))
    sb = S.astype(np.float16).view(np.uint8).reshape(-1)
    pk.scales.zero_()
    pk.scales[: sb.size].copy_(torch.from_numpy(sb))
    ZB = (G + 1) // 2
    zz = np.zeros((N, ZB * 2), np.uint8)
    zz[:, :G] = z
    zb = (zz[:, 0::2] | (zz[:, 1::2] << 4)).astype(np.uint8).reshape(-1)
    pk.zeros.zero_()
    pk.zeros[: zb.size].copy_(torch.from_numpy(zb))
    pk.svec[:K * 4].copy_(torch.from_numpy(np.ones(K, np.float32)).view(torch.uint8))
    return pk


def ref(codes_u8, S, z, x):
    N, K = codes_u8.shape
    G = K // 128
    Wd = (codes_u8.reshape(N, G, 128).astype(np.float64) - z[:, :, None]) * S.astype(np.float64)[:, :, None]
    return x.astype(np.float64) @ Wd.reshape(N, K).T


def run(N, K, codes, S, z, x, label):
    pk = make_packed(codes, S, z)
    xt = torch.from_numpy(x.astype(np.float16)).cuda()
    y = paro.paro_linear(xt, pk, flags=paro.PARO_LINEAR_NO_ROTATION).float().cpu().numpy()
    r = ref(codes, S, z, x.astype(np.float16))
    bad = np.abs(y - r) > 1e-2 * (1 + np.abs(r))
    print(f"[{label}] N={N} K={K} maxerr={np.max(np.abs(y - r)):.4g}  bad={bad.sum()}/{bad.size}")
    if bad.any():
        idx = np.argwhere(bad)[:8]
        for b, n in idx:
            print(f"   y[{b},{n}] gpu={y[b, n]:.5g} ref={r[b, n]:.5g}")
    return y, r


def main():
    torch.cuda.init()
    rng = np.random.default_rng(0)
    for (N, K) in [(256, 256), (64, 4096)]:
        G = K // 128
        ones = np.ones((N, K), np.uint8)
        S1 = np.ones((N, G), np.float16)
        z0 = np.zeros((N, G), np.uint8)
        run(N, K, ones, S1, z0, np.ones((1, K)), "all-ones")
        # one-hot x at several k: y[n] = q[n,k]
        codes = rng.integers(0, 16, size=(N, K)).astype(np.uint8)
        for k in [0, 1, 2, 3, 4, 5, 7, 8, 31, 32, 127, 128, K - 1]:
            x = np.zeros((1, K))
            x[0, k] = 1.0
            y, r = run(N, K, codes, S1, z0, x, f"onehot k={k}")
            if not np.allclose(y, r, atol=1e-2):
                # which code column did we pick up?
                for kk in range(min(K, 64)):
                    if np.allclose(y[0], codes[:, kk], atol=1e-2):
                        print(f"      -> matches code column {kk}")
        Sr = (rng.uniform(0.5, 2, size=(N, G))).astype(np.float16)
        zr = rng.integers(0, 16, size=(N, G)).astype(np.uint8)
        run(N, K, codes, Sr, zr, rng.normal(size=(1, K)), "random")
        run(N, K, codes, Sr, zr, rng.normal(size=(3, K)), "random B=3")
    # timing of q_proj without graph / PDL
    N, K = 4096, 4096
    G = K // 128
    pk = make_packed(rng.integers(0, 16, size=(N, K)).astype(np.uint8), np.ones((N, G), np.float16),
                     np.zeros((N, G), np.uint8))
    xt = torch.randn(1, K, device="cuda").half()
    y = paro.paro_linear(xt, pk, flags=paro.PARO_LINEAR_NO_ROTATION)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for flags, lab in [(paro.PARO_LINEAR_NO_ROTATION, "norot"), (0, "rot")]:
        for _ in range(10):
            paro.paro_linear(xt, pk, y=y, flags=flags)
        e0.record()
        for _ in range(100):
            paro.paro_linear(xt, pk, y=y, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        print(f"q_proj {lab}: {e0.elapsed_time(e1) / 100 * 1e3:.2f} us/call (eager, L2-warm)")


if __name__ == "__main__":
    main()
