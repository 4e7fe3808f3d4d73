"""Generate tests/golden/c5_oracle_samples.npz: the full-size C5 solution of the CPU oracle
(serial fp64 FMM, oracle/) at a seeded sample of gridpoints.

Run on a GPU box (the C5 speed field is evaluated with torch on the GPU exactly as the GPU
tests do, workloads.c5_field_torch); the arithmetic of the solution is oracle.fmm only --
nothing from the CUDA product path is imported.  ~15 min of serial CPU work at 1025^3.

    python tools/make_c5_golden.py            (writes tests/golden/c5_oracle_samples.npz + .json)

Recorded: SHA-256 of the fp64 F the oracle solved (and of its fp32 rounding, the array an fp32
GPU run receives), the exit list, the number of finite values, max U and where, and U at
  * 131072 points drawn with numpy default_rng(13064743).integers(0, M) (sorted, unique),
  * the 64 exits, the 8 grid corners, and the arg-max of U.
SURVEY 8(c) C.6 / 8(d) D.6 (cached C5 oracle run keyed by the F hash); VERDICT r1 item 1(b).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402

N = 1024
SAMPLE_SEED = 13064743
N_SAMPLES = 131072
OUT = os.path.join(ROOT, "tests", "golden", "c5_oracle_samples")


def c5_inputs_host(n: int = N, device: str = "cuda"):
    """The C5 input exactly as the GPU tests build it (fp64 F via torch on cuda:0)."""
    import torch
    a, c, sig, ex = W.c5_params(n)
    F64 = W.c5_field_torch(n, a, c, sig, device=device, dtype=torch.float64)
    F32h = F64.to(torch.float32).cpu().numpy()
    F64h = F64.cpu().numpy()
    del F64
    torch.cuda.empty_cache()
    return F64h, F32h, ex


def sample_index(M: int, ex, n: int):
    rng = np.random.default_rng(SAMPLE_SEED)
    idx = rng.integers(0, M, N_SAMPLES)
    n1 = n + 1
    extra = [i + n1 * (j + n1 * k) for (i, j, k) in ex]
    extra += [i + n1 * (j + n1 * k) for i in (0, n) for j in (0, n) for k in (0, n)]
    return np.unique(np.concatenate([idx.astype(np.int64), np.array(extra, dtype=np.int64)]))


def main():
    # dry run (CPU, reduced size, output elsewhere): make_c5_golden.py --n 64 --device cpu --out /tmp/x
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=N)
    ap.add_argument("--device", default="cuda")
    ap.add_argument("--out", default=OUT)
    args = ap.parse_args()
    n = args.n
    n1 = n + 1
    M = n1 ** 3
    t0 = time.time()
    F64, F32, ex = c5_inputs_host(n, args.device)
    h64 = hashlib.sha256(F64.tobytes()).hexdigest()
    h32 = hashlib.sha256(F32.tobytes()).hexdigest()
    del F32
    print(f"F generated and hashed in {time.time() - t0:.1f} s: {h64}", flush=True)
    mask = np.zeros(F64.shape, np.uint8)
    for (i, j, k) in ex:
        mask[k, j, i] = 1
    q = np.zeros(F64.shape, np.float64)
    oracle.build()
    t1 = time.time()
    U, cnt = oracle.fmm(n, F64, mask, q, return_count=True)
    t_fmm = time.time() - t1
    print(f"oracle FMM at {n1}^3: {t_fmm:.1f} s, {cnt} accepted", flush=True)
    Uf = U.reshape(-1)
    fin = np.isfinite(Uf)
    amax = int(np.argmax(np.where(fin, Uf, -1.0)))
    idx = np.unique(np.concatenate([sample_index(M, ex, n), np.array([amax], np.int64)]))
    np.savez_compressed(args.out + ".npz", idx=idx, U=Uf[idx])
    meta = {
        "what": "C5 (n=1024, 1025^3) fp64 FMM oracle values at sampled gridpoints",
        "generator": "tools/make_c5_golden.py (oracle.fmm on workloads.c5_field_torch(cuda, fp64))",
        "cites": "P:155-159 (FMM); BASELINE.json configs[4]; SURVEY 8(c) C.6, 8(d) D.6",
        "n": n, "M": M, "exits": [list(e) for e in ex],
        "F64_sha256": h64, "F32_sha256": h32,
        "n_finite": int(fin.sum()), "accepted": int(cnt),
        "U_max": float(Uf[amax]), "U_argmax": amax,
        "sample_seed": SAMPLE_SEED, "n_samples": int(idx.size),
        "oracle_seconds": round(t_fmm, 1),
    }
    json.dump(meta, open(args.out + ".json", "w"), indent=1)
    print(json.dumps({k: v for k, v in meta.items() if k != "exits"}), flush=True)


if __name__ == "__main__":
    main()
