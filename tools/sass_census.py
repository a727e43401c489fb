"""Static SASS opcode census of libpb_b200.so per kernel (cuobjdump -sass): evidence of the FP64
tensor path (DMMA.8x8x4), TMA bulk copies (UBLKCP) + mbarriers (SYNCS.*), cp.async (LDGSTS) staging,
L2 bulk prefetch (UBLKPF) and the shuffle / MUFU-based factorizations."""
import collections
import re
import subprocess
import sys

KEEP = ("DMMA", "UBLKCP", "UBLKPF", "SYNCS", "LDGSTS", "SHFL", "MUFU", "BAR.SYNC", "DFMA", "DMUL", "DADD")


def main(lib, out):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, counts = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P[0-9T] )?([A-Z0-9_.]+)", line)
        if cur and m:
            op = m.group(1)
            if op.startswith(KEEP):
                counts[cur][op] += 1
    lines = ["# static SASS opcode census of " + lib + " (tools/sass_census.py), per kernel.",
             "# DMMA.8x8x4 = mma.sync m8n8k4 f64 (tcgen05 has no f64 kind), UBLKCP = cp.async.bulk (TMA 1-D),",
             "# UBLKPF = cp.async.bulk.prefetch.L2, SYNCS.* = mbarrier, LDGSTS = cp.async, MUFU.RSQ64H = rsqrt seed."]
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    for (k, c), name in zip(counts.items(), names):
        name = name.replace("(anonymous namespace)::", "")[:120]
        lines.append(name)
        lines.append("    " + ", ".join(f"{op}:{n}" for op, n in sorted(c.items())))
    open(out, "w").write("\n".join(lines) + "\n")
    print(len(counts), "kernels")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
