"""Digest an ncu --set full --import-source report: headline metrics, opcode histogram and the hottest SASS
instructions by stall samples (usage: ncu_sass.py report.ncu-rep items_per_launch [top])."""
import collections
import csv
import io
import subprocess
import sys


def page(rep, which):
    out = subprocess.run(["ncu", "-i", rep, "--page", which, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, items, top=40):
    rows = page(rep, "raw")
    d = dict(zip(rows[0], rows[2]))
    for k in ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
              "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_registers",
              "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]:
        print(k, d.get(k))
    print("warp-instr/item", float(d["smsp__inst_executed.sum"]) / items)
    for k, v in d.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(v) > 0.15:
                    print("  ", k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v)
            except ValueError:
                pass
    rows = page(rep, "source")
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
    tot = sum(float(x["Instructions Executed"]) for x in data)
    ts = sum(float(x["# Samples"]) for x in data)
    byop, sop = collections.Counter(), collections.Counter()
    for x in data:
        w = x["Source"].split()
        op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
        byop[op] += float(x["Instructions Executed"])
        sop[op] += float(x["# Samples"])
    print(f"{len(data)} SASS instructions, {tot / items:.0f} warp-instr/item, {ts:.0f} samples")
    for op, c in byop.most_common(18):
        print(f"  {op:10s} {c / tot * 100:5.1f}% inst {sop[op] / ts * 100:5.1f}% samples {c / items:8.0f}/item")
    print("hottest instructions by samples:")
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for i, x in sorted(enumerate(data), key=lambda p: -float(p[1]["# Samples"]))[:top]:
        st = sorted(((float(x[c] or 0), c) for c in stall_cols), reverse=True)[:2]
        print(f"  #{i:5d} {float(x['# Samples']) / ts * 100:5.1f}% {float(x['Instructions Executed']) / items:7.1f}/item "
              f"{x['Source'][:70]:70s} {st[0][1]}={st[0][0]:.0f} {st[1][1]}={st[1][0]:.0f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
