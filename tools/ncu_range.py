"""Print the profiled SASS instructions attributed to a source line range (usage: ncu_range.py rep obj file lo hi)."""
import csv, glob, io, os, re, subprocess, sys, tempfile
rep, obj, fname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", glob.glob(tmp + "/*.cubin")[0]], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout)))
kname = rows[0][1]
short = re.sub(r"[<(].*", "", kname.replace("<unnamed>::", "")).split("::")[-1].split()[-1]
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
lines, cur, infn = [], ("?", 0), False
for ln in dis.splitlines():
    if ln.startswith("\t.section\t.text."):
        infn = short in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    elif re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
ts = sum(float(x["# Samples"]) for x in data)
scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
for i, (x, l) in enumerate(zip(data, lines)):
    if l[0] == fname and lo <= l[1] <= hi:
        s = float(x["# Samples"])
        tot += s
        st = sorted(((float(x[c] or 0), c[6:]) for c in scols), reverse=True)[:3]
        print(f"#{i:5d} L{l[1]:<4d} {s:6.0f} {float(x['Instructions Executed']):10.0f}  {x['Source'][:64]:64s} " + " ".join(f"{n}={v:.0f}" for v, n in st if v > 0))
print("range samples", tot, f"{tot / ts * 100:.1f}% of all")
