"""Write oracle slice values s_sigma for the committed plans (plans/<cfg>.json) to
tests/golden/parity_<cfg>.json.

Imports ONLY oracle/ and circuits/ (the seeded input generators): no value here comes from the
CUDA path.  s_sigma is Eq. sliced_sum's partial sum of the sigma-restricted
network contracted along the plan's SSA path (Eq. seq, l.95-105), in complex128.

Slice picks: one seeded slice in each of the G=8 contiguous rank blocks
of the canonical slice order (block 0 contributes slice 0), or an explicit list.

  python scripts/make_goldens.py C3 [--per-block 1] [--blocks 8] [--extra i,j]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from circuits import workload  # noqa: E402
from circuits.rng import SplitMix64  # noqa: E402
from oracle import contract, cost  # noqa: E402
from oracle.network import build_network  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def picks_for(n_sl, blocks, per_block, seed):
    rng = SplitMix64(seed)
    out = []
    for g in range(blocks):
        b, e = g * n_sl // blocks, (g + 1) * n_sl // blocks
        for q in range(per_block):
            if g == 0 and q == 0:
                out.append(b)
            else:
                out.append(b + int(rng.next_u64() % (e - b)))
    return sorted(set(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--per-block", type=int, default=1)
    ap.add_argument("--indices", default="")
    ap.add_argument("--seed", type=int, default=2107)
    args = ap.parse_args()
    plan = json.load(open(os.path.join(ROOT, "plans", f"{args.config}.json")))
    circ, bits = workload(plan["circuit"], plan["circuit_seed"])
    net = build_network(circ, bits)
    path = [tuple(s) for s in plan["ssa_path"]]
    sl = list(plan["sliced_labels"])
    steps = cost.tree_info(net, path, sl)       # (cost_report would enumerate all N_sl slices)
    rep = {"flop_sl": sum(f for f, _ in steps)}
    n_sl = 1
    for l in sl:
        n_sl *= net.dims[l]
    if args.indices:
        idx = sorted(int(x) for x in args.indices.split(","))
    else:
        idx = picks_for(n_sl, min(args.blocks, n_sl), args.per_block, args.seed)
    out_path = os.path.join(ROOT, "tests", "golden", f"parity_{args.config}.json")
    old = json.load(open(out_path)) if os.path.exists(out_path) else {}
    same = old.get("plan_sha") == plan_sha(plan) and old.get("bitstring", list(bits)) == [int(b) for b in bits]
    slices = {int(k): v for k, v in old.get("slices", {}).items()} if same else {}
    def write():
        rec = {
            "config": args.config, "plan": f"plans/{args.config}.json", "plan_sha": plan_sha(plan),
            "bitstring": [int(b) for b in bits],
            "what": "oracle s_sigma (complex128 numpy, oracle/contract.py) of the sigma-restricted network "
                    "along the plan's SSA path; PAPER.md l.95-105 (Eq. seq), l.123-128 (Eq. sliced_sum)",
            "script": "scripts/make_goldens.py (imports only oracle/ and circuits/)",
            "n_sl": n_sl, "flop_sl": rep["flop_sl"], "blocks": args.blocks,
            "host": {"cpu_model": cpu_model(), "threads": blas_threads(), "nproc": os.cpu_count()},
            "slices": {str(k): slices[k] for k in sorted(slices)},
        }
        with open(out_path, "w") as f:
            json.dump(rec, f, indent=1)

    for i in idx:
        if i in slices:
            continue
        t0 = time.perf_counter()
        (v,) = contract.slice_values(net, path, sl, indices=[i])
        dt = time.perf_counter() - t0
        slices[i] = {"re": v.real, "im": v.imag, "oracle_s": round(dt, 2)}
        import resource
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
        print(f"{args.config} slice {i}: {v!r} ({dt:.1f} s, max rss {rss:.1f} GB)", flush=True)
        write()
    write()


def plan_sha(plan):
    import hashlib

    s = json.dumps({"p": plan["ssa_path"], "s": plan["sliced_labels"], "c": plan["circuit"],
                    "seed": plan["circuit_seed"]}, sort_keys=True)
    return hashlib.sha256(s.encode()).hexdigest()[:16]


if __name__ == "__main__":
    main()
