"""Evaluate planner settings on a workload: prefix-cache FLOP / bytes and roofline time."""
import sys, time
sys.path.insert(0, '.')
from circuits import workload
from paper_2107_09793_b200 import jet

def evaluate(plan, dtype="c64"):
    d = plan.describe_exec(dtype)
    tb = tf = 0
    for n in d['nodes']:
        runs = 2 ** (n['maxpos'] + 1)
        tb += n['bytes'] * runs
        tf += n['flop'] * runs
    return tf, tb, d['total_bytes']

if __name__ == "__main__":
    name = sys.argv[1]; k = int(sys.argv[2])
    c, x = workload(name)
    net = jet.Network.from_circuit(c, x)
    for R in [float(r) for r in sys.argv[3].split(",")]:
        for trials in [int(t) for t in sys.argv[4].split(",")]:
            for cands in [int(t) for t in sys.argv[5].split(",")]:
                t = time.time()
                g = jet.Plan.greedy(net, seed=1, trials=trials, n_sliced=k, bytes_weight=R, candidates=cands)
                dt = time.time() - t
                tf, tb, ws = evaluate(g)
                co = g.cost()
                print("R=%g trials=%d cand=%d: flop %.3g bytes %.3g width %d t_hbm=%.1fs t_fp32=%.1fs t_tc=%.1fs ws=%.0fGB plan %.1fs" % (
                    R, trials, cands, tf, tb, co['max_width'], tb / 6.5e12, tf / 70e12, max(tb/6.5e12, tf/300e12), ws / 1e9, dt), flush=True)
