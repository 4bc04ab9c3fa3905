"""Diagnostic: iteration-1..3 deviation of the world-size-2 hosted sharded run
from the single-GPU run over a sweep of shapes."""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_hosted_sharded as T  # noqa: E402

SWEEP = {
    "a": (300, 241, 2, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
    "b": (300, 240, 2, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
    "c": (300, 241, 2, 0, 1, 0.01, 8, 12, 1, 3, 1, True),
    "d": (300, 241, 8, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
    "e": (1000, 1001, 2, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
    "f": (300, 241, 2, 0, 1, 0.01, 8, 12, 0, 3, 1, False),
    "g": (300, 241, 2, 0, 1, 0.01, 4, 12, 1, 3, 1, False),
    "h": (300, 241, 20, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
    "i": (1000, 1001, 20, 0, 1, 0.01, 8, 12, 1, 3, 1, False),
}


def main():
    import socket

    import torch.multiprocessing as mp

    import paper_1712_02248_b200 as cb
    T.CASES.update(SWEEP)
    ctx = cb.Context(0)
    for case in SWEEP:
        d, n, r, fk, nk, sigma, k, q, w, iters, every, stream = T.CASES[case]
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        with tempfile.TemporaryDirectory() as tmp:
            mp.start_processes(T._worker, args=(2, port, SWEEP[case], tmp), nprocs=2, join=True,
                               start_method="spawn")
            res = np.load(os.path.join(tmp, "rank0.npz"))
        if stream:
            os.environ["CNMF_HALS"] = "stream"
        xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
        ctx.synth_x(d, n, r, fk, nk, sigma, 1, xb)
        a1, b1, t1 = ctx.run_device(xb[:, :n], T._cfg(cb, k, q, w, iters, every))
        os.environ.pop("CNMF_HALS", None)
        e1 = np.array([z.error for z in t1.records])
        dev = np.abs(res["err"] - e1) / e1
        print(case, SWEEP[case][:9], " ".join(f"{v:.1e}" for v in dev), "redraws", t1.redraws,
              int(res["redraws"][0]), flush=True)


if __name__ == "__main__":
    main()
