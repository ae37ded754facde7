"""Full-size parity fixtures for the five BASELINE configs (TEST INFRASTRUCTURE).

Runs on a GPU box (the inputs are generated on the device, deterministically:
matgen.device_input with QDWHG_FLAG_DETERMINISTIC, so the bytes and their
SHA-256 are reproducible on every B200).  For each config it copies A to the
host, hashes it, and runs the CPU oracle on those exact bytes:

  * the numpy restatement (oracle/qdwh_oracle.py, pinned against the reference's
    own outputs by tests/test_oracle_pins.py) with all host threads, and
  * with --ref, the reference ITSELF (oracle/_ref/libqdwhref.so, single thread)
    — the same-input reference time-to-solution reported by bench.py.

    python tests/golden/make_fullsize.py --cfg 1 2 3 4 5 [--ref 1 2] [--out DIR]

Output: DIR/cfgN.npz with the input hash, the request (shift c / cut), the
oracle's top-k values (k by count, BASELINE.json's k), its ell / ind /
iteration counts / mu or alpha, and the wall times.  The committed copies live
in tests/golden/fullsize/ and are read by tests/test_gpu_fullsize.py and bench.py.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def oracle_solve(inp, a):
    """Run the numpy oracle on host bytes `a`; returns (top-k values, meta)."""
    from oracle import qdwh_oracle as O
    k = inp["k"]
    t0 = time.perf_counter()
    if inp["kind"] == "eig":
        n = a.shape[0]
        b = inp["c"] * np.eye(n) - a
        r = O.qdwh_partial_eig(b, O.choose_shift(3))
        dt = time.perf_counter() - t0
        vals = inp["c"] - r.lambda_minus[:k]  # largest first
        meta = dict(found=r.count(), ell=r.subspace_size, ind=r.rank_index, mu=r.mu,
                    iters_chol=r.iters_chol, iters_qr=r.iters_qr)
    else:
        alpha = O.two_norm_estimate(a)
        r = O.qdwh_partial_svd(a, inp["cut"] / alpha, use_randomization=bool(inp.get("randomize")))
        dt = time.perf_counter() - t0
        vals = r.sigma1[:k]
        meta = dict(found=r.count(), ell=r.subspace_size, ind=r.rank_index, alpha=r.alpha,
                    iters_chol=r.iters_chol, iters_qr=r.iters_qr)
    meta["seconds"] = dt
    return np.asarray(vals, dtype=np.float64), meta


def reference_solve(inp, a):
    """The reference itself (single-threaded C++) on host bytes `a`."""
    from oracle import ref as R
    k = inp["k"]
    t0 = time.perf_counter()
    if inp["kind"] == "eig":
        n = a.shape[0]
        lam, _, d = R.partial_eig(inp["c"] * np.eye(n) - a, 3)
        dt = time.perf_counter() - t0
        vals = inp["c"] - np.asarray(lam)[:k]
    else:
        alpha = R.two_norm_estimate(a)
        sig, _, _, d = R.partial_svd(a, inp["cut"] / alpha, randomize=bool(inp.get("randomize")))
        dt = time.perf_counter() - t0
        vals = np.asarray(sig)[:k]
    return np.asarray(vals, dtype=np.float64), dict(seconds=dt, ell=d["subspace_size"],
                                                    found=len(vals))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    import torch
    from paper_2104_14186_b200 import matgen
    p = argparse.ArgumentParser()
    p.add_argument("--cfg", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    p.add_argument("--ref", type=int, nargs="*", default=[])
    p.add_argument("--out", default=os.path.join(HERE, "fullsize"))
    args = p.parse_args()
    os.makedirs(args.out, exist_ok=True)
    dev = torch.device("cuda", 0)
    for cfg in args.cfg:
        t0 = time.perf_counter()
        inp = matgen.device_input(cfg, dev)
        torch.cuda.synchronize()
        a = matgen.host_copy(inp["A"])
        del inp["A"]
        torch.cuda.empty_cache()
        sha = matgen.input_sha256(a)
        tgen = time.perf_counter() - t0
        vals, meta = oracle_solve(inp, a)
        rec = dict(cfg=cfg, sha256=sha, k=inp["k"], kind=inp["kind"],
                   request=inp.get("c", inp.get("cut")), randomize=bool(inp.get("randomize", False)),
                   values=vals, oracle=json.dumps(meta), gen_seconds=tgen,
                   host_cpu=cpu_model(), host_threads=os.cpu_count())
        if cfg in args.ref:
            rv, rmeta = reference_solve(inp, a)
            rec["ref_values"] = rv
            rec["reference"] = json.dumps(rmeta)
            print(f"cfg{cfg}: reference {rmeta['seconds']:.1f} s, max rel vs oracle "
                  f"{np.max(np.abs(rv - vals) / np.abs(vals)):.2e}", flush=True)
        np.savez_compressed(os.path.join(args.out, f"cfg{cfg}.npz"), **rec)
        print(f"cfg{cfg}: sha {sha[:16]} k={inp['k']} oracle {meta}", flush=True)
        del a


if __name__ == "__main__":
    main()
