"""Depth-slab plan of the engine at a config for N = 2, 4, 8 ranks (created
one rank at a time on this GPU with a no-op all-reduce; nothing runs): per
rank the z-planes, voxels, active samples (the DAS work), the RF sample
window it reads and its host -> device RF bytes per ensemble, plus the
NVLink-broadcast alternative (one upload of the union window on rank 0).

    python scripts/shard_plan.py C
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05464_b200 import workloads as W  # noqa: E402
from paper_2509_05464_b200.engine import Engine  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C"
    w = W.config(cfg)
    F, A, T, E = w.rf_shape()
    out = {"config": cfg, "full_rf_bytes": 4 * F * A * T * E}
    for n in (1, 2, 4, 8):
        ranks = []
        for r in range(n):
            eng = Engine(w.fs, 0.0, w.angles, F, T, w.grid, w.elements, w.bf(), rank=r, world=n,
                         allreduce=(lambda *a: 0) if n > 1 else None)
            i = eng.info
            ranks.append({"rank": r, "planes": [i.k_begin, i.k_end],
                          "voxels": int(i.v_end - i.v_begin),
                          "active_samples": int(i.active_samples),
                          "rf_window": [i.t_begin, i.t_end],
                          "h2d_bytes": int(i.h2d_bytes_per_ensemble),
                          "device_gb": round(i.device_bytes / 1e9, 2)})
            eng.close()
        act = [x["active_samples"] for x in ranks]
        tb = min(x["rf_window"][0] for x in ranks)
        te = max(x["rf_window"][1] for x in ranks)
        out[f"N={n}"] = {"ranks": ranks,
                         "h2d_total_per_ensemble": sum(x["h2d_bytes"] for x in ranks),
                         "h2d_broadcast_mode": 4 * F * A * (te - tb) * E,
                         "das_balance_max_over_mean": max(act) / (sum(act) / n)}
        print(json.dumps({"N": n, **out[f"N={n}"]}), flush=True)
    json.dump(out, open(os.path.join("gpurun_out", f"shard_plan_{cfg}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
