"""Time the workload generator (device cut-cell quadrature vs host) on a BASELINE config."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import classify, generate  # noqa: E402
from workloads import config_voids, get_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = get_config(name)
c, r = config_voids(cfg)
t0 = time.time()
kind, ncut = classify(cfg, c, r)
t1 = time.time()
G = generate(cfg, c, r, kind=kind, device=True)
t2 = time.time()
out = {"config": name, "n_cut": int(ncut), "classify_s": t1 - t0, "device_gen_s": t2 - t1}
if len(sys.argv) > 2:   # host comparison on a sample
    k = int(sys.argv[2])
    s = G.cut_cells[:: max(1, len(G.cut_cells) // k)][:k]
    t3 = time.time()
    H = generate(cfg, c, r, kind=kind, cut_cells=s, device=False)
    t4 = time.time()
    idx = np.searchsorted(G.cut_cells, s)
    err = np.sqrt(((H.cut_K - G.cut_K[idx]) ** 2).sum(axis=(1, 2)) / (H.cut_K ** 2).sum(axis=(1, 2))).max()
    out.update({"host_sample": int(len(s)), "host_sample_s": t4 - t3,
                "host_full_est_s": (t4 - t3) * ncut / len(s), "max_rel_diff": float(err)})
print(json.dumps(out))
