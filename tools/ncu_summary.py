"""One-line-per-kernel summary of an ncu --set full report (raw page): duration, DRAM bytes,
throughputs, tensor-pipe activity, occupancy, top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "dur_ns"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
        ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")[:70]
        vals = []
        for k, lab in KEYS:
            if k in d:
                vals.append(f"{lab}={d[k]}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        top = ", ".join(f"{n} {s / tot:.0%}" for s, n in stalls[:5])
        print(f"{name}\n    " + " ".join(vals) + f"\n    stalls: {top}")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        main(rep)
