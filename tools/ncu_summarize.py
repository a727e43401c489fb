"""Summarise ncu --set full reports of the C2 potrf kernels (run where the .ncu-rep files are)."""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
ITEMS = {8: 10066330, 16: 2516583, 32: 524288, 64: 98304, 128: 24576}


def main(prefix, out):
    lines = ["# ncu --set full --clock-control none, one launch per C2 point (bench.py --only 'potrf_l n=N'), "
             "current kernels, B200",
             "# n | kernel | grid x block | regs | ms | DRAM rd+wr B/item | DRAM % peak | warps active % | "
             "issue active % | warp-instr/item | fp64 pipe %"]
    for n, it in ITEMS.items():
        r = subprocess.run(["ncu", "-i", f"{prefix}{n}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                           text=True).stdout
        rows = list(csv.reader(io.StringIO(r)))
        if len(rows) < 3:
            lines.append(f"{n} | (no report)")
            continue
        d = dict(zip(rows[0], rows[2]))
        b = (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * 1e9 / it
        lines.append(f"{n} | {d['Kernel Name'][:52]} | {d['launch__grid_size']}x{d['launch__block_size']} | "
                     f"{d['launch__registers_per_thread']} | {float(d['gpu__time_duration.sum']):.3f} | {b:.0f} | "
                     f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{float(d['smsp__inst_executed.sum']) / it:.0f} | "
                     f"{float(d['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']):.1f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
