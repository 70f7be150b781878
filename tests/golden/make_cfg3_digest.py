"""Digest of the C oracle's full cfg3 sweep (K = 150), for the GPU test
tests/test_gpu_large.py::test_cfg3_full_k_bitwise_vs_oracle_digest.

The oracle (oracle/fsda_oracle.c, the device's summation order, deferred
shift-update mode 2) takes minutes per cfg3 solve on the host, so the GPU
box compares against this committed sha256 instead of re-running it.  The
workload digest pins the generator's arrays.

    python tests/golden/make_cfg3_digest.py     # writes tests/golden/cfg3_oracle_digest.json
"""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import c_oracle  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload, workload_digest  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    w = make_workload("cfg3")
    c_oracle.build()
    c_oracle.set_shift_mode(2)
    t0 = time.time()
    ref = c_oracle.fsda_solve_workload(w)
    out = {
        "workload": "cfg3", "workload_sha256": workload_digest(w), "max_iter": w.max_iter,
        "shift_update_mode": 2,
        "directions_sha256": sha(ref["directions"]), "scores_sha256": sha(ref["scores"]),
        "residuals_sha256": sha(ref["residuals"]), "iterations": ref["iterations"].tolist(),
        "converged": ref["converged"].astype(int).tolist(), "n_applies": int(ref["n_applies"]),
        "direction_norms": np.linalg.norm(ref["directions"], axis=1).tolist(),
        "oracle_seconds": time.time() - t0,
    }
    (Path(__file__).parent / "cfg3_oracle_digest.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: v for k, v in out.items() if "sha" in k or k == "oracle_seconds"}))


if __name__ == "__main__":
    main()
