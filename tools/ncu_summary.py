"""Per-kernel summary of an `ncu --set full` report: duration, DRAM bytes, tensor-pipe and
SM throughput, achieved occupancy. Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "bytes"),
    ("dram__bytes_write.sum", "bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("launch__registers_per_thread", ""),
    ("sm__cycles_elapsed.avg.per_second", "GHz"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "bytes"),
]


def to_base(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-3, "usecond": 1,
             "msecond": 1e3, "us": 1, "ns": 1e-3, "ms": 1e3}
    return v * scale.get(unit, 1)


def main(path, json_out=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    traffic = {}
    print("| kernel | " + " | ".join(m.split(".")[0] + f" ({u})" for m, u in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0][-60:]
        vals = []
        for m, u in METRICS:
            if m not in h:
                vals.append("-")
                continue
            i = h.index(m)
            v = to_base(r[i], units[i]) if r[i] not in ("", "n/a") else float("nan")
            vals.append(f"{v / 1e6:.1f} MB" if u == "bytes" else f"{v:.1f}")
        print(f"| {name} | " + " | ".join(vals) + " |")
        rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        traffic[name.strip()] = {"dram_bytes": to_base(r[rd], units[rd]) + to_base(r[wr], units[wr]),
                                 "duration_us": to_base(r[h.index("gpu__time_duration.sum")],
                                                        units[h.index("gpu__time_duration.sum")])}
    if json_out:
        import json
        with open(json_out, "w") as f:
            json.dump({"source": path, "kernels": traffic}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
