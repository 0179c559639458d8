"""Per-source-line warp-stall attribution of one ncu capture: join the SASS source page
(ncu -i rep --page source --csv --print-source sass) with nvdisasm --print-line-info of the
kernel in libjetb200.so (the ncu page lists SASS without line info).

  python scripts/ncu_lines.py <source.csv> <mangled kernel name> [top] [nvdisasm output of the
  profiled build] [csrc directory of the profiled build] (the last two when the current
  libjetb200.so is a later build)"""
import collections, csv, os, re, subprocess, sys, tempfile

src_csv, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_2107_09793_b200", "libjetb200.so")
dis = open(sys.argv[4]).read() if len(sys.argv) > 4 else None
if dis is None:
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True)
        dis = ""
        for f in os.listdir(td):
            if not f.endswith(".cubin"):
                continue
            r = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(td, f)], capture_output=True, text=True)
            if ".text." + kname + ":" in r.stdout:
                dis = r.stdout
lines, cur, on = {}, None, False
for l in dis.split("\n"):
    if l.startswith(".text." + kname + ":"):
        on = True
        continue
    if on and l.startswith(".text."):
        break
    if not on:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*)", l)
    if m:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
tot, per, stl = 0, collections.Counter(), collections.defaultdict(collections.Counter)
for r in data:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ln = lines.get(int(r[0], 16) - base)
    tot += n
    per[ln] += n
    for s in stalls:
        stl[ln][s] += int(r[ix[s]] or 0)
srcs = {}
for ln in per:
    if ln and ln[0] not in srcs:
        csrc = sys.argv[5] if len(sys.argv) > 5 else os.path.join(root, "paper_2107_09793_b200", "csrc")
        p = os.path.join(csrc, ln[0])
        srcs[ln[0]] = open(p).read().split("\n") if os.path.exists(p) else []
print(f"# {kname}: {tot} warp-stall samples; share, file:line, top stall reasons, source")
for ln, n in per.most_common(top):
    txt = srcs.get(ln[0], [])[ln[1] - 1].strip()[:80] if ln and srcs.get(ln[0]) else ""
    why = ", ".join(f"{k[6:]} {v / max(n, 1):.0%}" for k, v in stl[ln].most_common(2))
    print(f"{100 * n / tot:6.2f}%  {ln[0] if ln else '?'}:{ln[1] if ln else 0}  [{why}]  {txt}")
