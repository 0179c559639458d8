"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch)."""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    h = rows[hi]
    ki, mi, vi, ii, gi, bi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID', 'Grid Size', 'Block Size'))
    per = collections.defaultdict(dict); meta = {}
    for r in rows[hi + 1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(',', ''))
        meta[int(r[ii])] = (r[ki], r[gi], r[bi])
    return per, meta

if __name__ == "__main__":
    per, meta = load(sys.argv[1])
    tot = collections.defaultdict(float); cnt = collections.Counter(); byt = collections.defaultdict(float)
    for i, m in per.items():
        n = meta[i][0].split('(')[0]
        tot[n] += m['gpu__time_duration.sum']; cnt[n] += 1
        byt[n] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    T = sum(tot.values())
    print("kernel, launches, total_ms, share, dram_GBps")
    for n in sorted(tot, key=lambda x: -tot[x]):
        print("%s, %d, %.3f, %.1f%%, %.0f" % (n, cnt[n], tot[n] / 1e6, 100 * tot[n] / T, byt[n] / tot[n]))
    big = sorted(per.items(), key=lambda x: -x[1]['gpu__time_duration.sum'])[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]
    print("top launches: id, kernel, grid, block, ms, dram GB/s, read GB, write GB")
    for i, m in big:
        t = m['gpu__time_duration.sum']; rd = m.get('dram__bytes_read.sum', 0); wr = m.get('dram__bytes_write.sum', 0)
        print("%d, %s, %s, %s, %.3f, %.0f, %.3f, %.3f" % (i, meta[i][0].split('(')[0], meta[i][1], meta[i][2], t / 1e6, (rd + wr) / t, rd / 1e9, wr / 1e9))
