"""Summarise an ncu report (raw page) per kernel: time, DRAM bytes, achieved
bandwidth, occupancy, issue rate, pipe utilisation and top stall reasons.
  python tools/ncu_summary.py gpurun_out/X.ncu-rep [edges_per_launch]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}

    def g(r, k, default=0.0):
        i = col.get(k)
        if i is None or r[i] in ("", "n/a"):
            return default
        try:
            return float(r[i].replace(",", ""))
        except ValueError:
            return r[i]

    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("esg::", "").replace("(anonymous namespace)::", "")
        t_ms = g(r, "gpu__time_duration.sum")
        if units[col["gpu__time_duration.sum"]] == "us":
            t_ms /= 1e3
        elif units[col["gpu__time_duration.sum"]] == "ns":
            t_ms /= 1e6
        def gb(k):
            v = g(r, k)
            u = units[col[k]] if k in col else ""
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(u, 1)
        rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
        print(f"{short[:60]:60s} grid {r[col['Grid Size']]} block {r[col['Block Size']]}")
        print(f"   time {t_ms:.3f} ms  dram rd {rd/1e9:.3f} GB wr {wr/1e9:.3f} GB  -> {(rd+wr)/t_ms/1e6:.0f} GB/s")
        print(f"   regs {g(r,'launch__registers_per_thread'):.0f}  warps active {g(r,'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%"
              f"  IPC/SM {g(r,'sm__inst_executed.avg.per_cycle_active'):.2f}"
              f"  fma {g(r,'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%"
              f"  tensor {g(r,'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%"
              f"  L2 hit {g(r,'lts__t_sector_hit_rate.pct'):.1f}%  L1 hit {g(r,'l1tex__t_sector_hit_rate.pct'):.1f}%")
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                st.append((g(r, k), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        st.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
