"""Attribute an ncu source-page (SASS) report to CUDA source lines through nvdisasm -g line markers.
usage: ncu_lines.py report.ncu-rep object.o items_per_launch [top]   (object.o built with -lineinfo)"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, items, top=40, kern=None):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kname = rows[0][1]
    short = re.sub(r"[<(].*", "", kname.replace("<unnamed>::", "")).split("::")[-1].split()[-1]
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
    # walk the disassembly of the matching function
    lines, cur, infn = [], ("?", 0), False
    for ln in dis.splitlines():
        if ln.startswith("\t.section\t.text."):
            infn = short in ln and (kern is None or kern in ln)
            continue
        if not infn:
            continue
        m = re.search(r'//## File "(.*)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            lines.append(cur)
    if len(lines) != len(data):
        print(f"warning: {len(lines)} disassembled vs {len(data)} profiled instructions ({short}); trying by kernel name")
    n = min(len(lines), len(data))
    inst, smp = collections.Counter(), collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for i in range(n):
        inst[lines[i]] += float(data[i]["Instructions Executed"])
        smp[lines[i]] += float(data[i]["# Samples"])
        for c in scols:
            stall[lines[i]][c] += float(data[i][c] or 0)
    ti, ts = sum(inst.values()), sum(smp.values())
    print(f"{kname[:80]}: {ti / items:.0f} warp-instr/item, {ts:.0f} samples")
    src = {}
    for k in sorted(smp, key=lambda k: -smp[k])[:top]:
        f, l = k
        if f not in src:
            p = [q for q in glob.glob("paper_1704_02457_b200/csrc/*") if os.path.basename(q) == f]
            src[f] = open(p[0]).read().splitlines() if p else []
        text = src[f][l - 1].strip()[:70] if 0 < l <= len(src[f]) else ""
        st = ", ".join(f"{c[6:]}={v / max(smp[k], 1) * 100:.0f}%" for c, v in stall[k].most_common(2))
        print(f"{smp[k] / ts * 100:5.1f}% smp {inst[k] / items:7.0f} ins/item  {f}:{l:<4d} {text:70s} [{st}]")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
