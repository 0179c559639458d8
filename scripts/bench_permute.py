"""K1 bit-permutation bandwidth on one B200 (target >= 70% of HBM peak on
>= 2^26-element tensors).  Algorithmic bytes = 2 * 2^n * esize per launch; CUDA events on
the launching stream; inputs larger than L2 (>= 512 MiB)."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2107_09793_b200 import jet  # noqa: E402


def perms(n, rng):
    yield "reverse", list(reversed(range(n)))
    yield "random", [int(x) for x in rng.permutation(n)]
    yield "rotate_low8", list(range(8, n)) + list(range(8))
    yield "swap_low_high", list(range(n - 4, n)) + list(range(4, n - 4)) + list(range(4))
    yield "identity", list(range(n))


def main():
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    import bench

    rng = np.random.default_rng(1)
    out = []
    clk = bench.ClockSampler(torch.cuda.current_device())
    clk.start()
    for dt, tdt in (("c64", torch.complex64), ("c128", torch.complex128)):
        for n in (26, 28):
            src = torch.randn(1 << n, dtype=tdt, device="cuda")
            dst = torch.empty_like(src)
            for name, perm in perms(n, rng):
                for _ in range(3):
                    jet.permute(src, perm, out=dst)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 10
                torch.cuda.synchronize()
                s.record()
                for _ in range(reps):
                    jet.permute(src, perm, out=dst)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / reps
                gbs = 2 * (1 << n) * src.element_size() / (ms / 1e3) / 1e9
                out.append({"dtype": dt, "n_bits": n, "perm": name, "ms": ms, "GBps": gbs, "frac_of_measured_hbm": gbs / peak})
                print(json.dumps(out[-1]), flush=True)
    clocks = clk.stop()
    print(json.dumps({"summary": "K1 permute", "peak_gbs_measured": peak, "clocks": clocks,
                      "min_frac": min(o["frac_of_measured_hbm"] for o in out if o["perm"] != "identity"),
                      "median_frac": float(np.median([o["frac_of_measured_hbm"] for o in out]))}))


if __name__ == "__main__":
    main()
