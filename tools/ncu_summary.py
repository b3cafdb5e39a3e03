"""Summarise an ncu report: key raw metrics, stall reasons, hottest SASS.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass 25]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 25
    hdr, rows = raw(rep)
    for row in rows:
        print("kernel:", row[hdr.index("Kernel Name")][:100])
        for k in KEYS:
            if k in hdr:
                print(f"  {k:72s} {row[hdr.index(k)]}")
        st = []
        for i, h in enumerate(hdr):
            if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
                try:
                    st.append((float(row[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("  stalls:", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, isamp = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return None
    data = [r for r in rows[2:] if len(r) > isamp and f(r[isamp]) is not None]
    tot = sum(f(r[isamp]) for r in data) or 1
    print(f"  sass: {len(data)} instructions, {tot:.0f} samples")
    for r in sorted(data, key=lambda r: -f(r[isamp]))[:nsass]:
        print(f"  {100 * f(r[isamp]) / tot:5.1f}% ex={r[iex]:>8s} {r[isrc][:90]}")


if __name__ == "__main__":
    main()
