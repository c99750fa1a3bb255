"""Trace of the whole BASELINE configs[0] (C1) optimisation run on the oracle,
for the north star's mask criterion (tests/test_gpu_c1_masks.py):

    python tests/golden/make_c1_trace.py

C1: 40x20x20 cantilever, E = 1, nu = 0.3, void 1e-3, x = 0 clamped, nodal
force (0, 0, -1) at node (40, 10, 10), compliance <= 1.6 J0, 4^3
agglomerates, PCG tolerance 1e-8, the SPEC's volume schedule (oracle
defaults). The oracle's loop is the SPEC restated
(oracle/topovox_oracle.py run_optimizer; the reference has no optimizer
code) over the oracle's FEA, which is pinned to the reference's golden
vectors.

Recorded for every extraction of the run (outer step k, inner iteration it):
the topology the fields were computed on (bit-packed), the AL weights, the
target volume fraction, the threshold tau, the extracted mask (bit-packed),
max|levelset|, the level-set values of every element within 1e-6 max|ls| of
tau (the near-threshold set) and at 256 fixed sample elements; plus the
run's final mask, per-outer history and stop reason.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from oracle import topovox_oracle as O  # noqa: E402

OUT = os.path.join(HERE, "c1_trace.npz")
NX, NY, NZ = 40, 20, 20
LOAD = (40, 10, 10)


def main():
    from conftest import cantilever

    d, case, fixed, f = cantilever(NX, NY, NZ, LOAD, LOAD)
    sample = np.sort(np.random.default_rng(99).choice(d.n_elems, 256, replace=False))
    recs = []

    def trace(r):
        ls = r["levelset"]
        m = float(np.abs(ls).max())
        near = np.flatnonzero(np.abs(ls - r["tau"]) <= 1e-6 * m)
        recs.append(dict(k=r["k"], it=r["it"], occ=np.packbits(r["occ"] == 1.0), w=np.array(r["weights"]),
                         target=r["target"], tau=r["tau"], new=np.packbits(r["new_occ"] == 1.0), maxabs=m,
                         near_idx=near.astype(np.int32), near_val=ls[near], sample_val=ls[sample]))
        print(f"  step k={r['k']} it={r['it']} target={r['target']:.4f} tau={r['tau']:.6g} near={near.size}",
              flush=True)

    t0 = time.time()
    occ, hist, reason = O.run_optimizer(NX, NY, NZ, [(fixed, f)], [{"kind": "compliance", "alpha": 1.6, "case": 0}],
                                        block=4, ersatz=1e-3, tol=1e-8, trace=trace)
    print(f"oracle C1 run: {len(hist)} outer steps, {len(recs)} extractions, {reason}, "
          f"final volume {np.mean(occ == 1.0):.4f}, {time.time() - t0:.0f} s", flush=True)
    out = {"sample": sample, "reason": np.array(reason), "final": np.packbits(occ == 1.0),
           "hist_v": np.array([h["v"] for h in hist]), "hist_acc": np.array([h["accepted"] for h in hist]),
           "hist_J": np.array([h["J"] for h in hist]), "n": np.int64(len(recs)), "seconds": time.time() - t0}
    for i, r in enumerate(recs):
        for key, v in r.items():
            out[f"s{i}_{key}"] = np.asarray(v)
    np.savez_compressed(OUT, **out)


if __name__ == "__main__":
    main()
