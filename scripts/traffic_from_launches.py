"""profiles/traffic.json from an ncu launch list (dram__bytes_read.sum + dram__bytes_write.sum per
launch), per config and kernel class (K3 = gett_tc_kernel, K3G = gett_tcg_kernel, K2 = gett_kernel,
K4 = gett_dmma_kernel, K2S = stream_gett_kernel, K1G = view_gather_kernel: the K1 copies feeding K3g)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launches import load

csv_path, cfg = sys.argv[1], sys.argv[2]
per, meta = load(csv_path)
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(out_path)) if os.path.exists(out_path) else {}
entry = {}
for cls, pat in (("K3", "gett_tc_kernel"), ("K3G", "gett_tcg_kernel"), ("K2", "gett_kernel<"), ("K4", "gett_dmma"),
                 ("K2S", "stream_gett_kernel"), ("K1G", "view_gather_kernel")):
    ls = [m for i, m in per.items() if pat in meta[i][0]]
    if not ls:
        continue
    tot_t = sum(m["gpu__time_duration.sum"] for m in ls)
    tot_b = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ls)
    entry[cls] = {"launches": len(ls), "dram_bytes_per_launch": tot_b / len(ls),
                  "dram_GBps_serialised": tot_b / tot_t, "source": os.path.basename(csv_path)}
d[cfg] = entry
json.dump(d, open(out_path, "w"), indent=1)
print(json.dumps(d, indent=1))
