"""One line per kernel launch of an .ncu-rep: time, DRAM bytes, achieved GB/s, pipe utilisation.
Usage: python tools/ncu_table.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def main(path, title=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]

    def val(r, k):
        return float(r[hdr.index(k)].replace(",", ""))

    def mb(r, k):
        return val(r, k) * SCALE[units[hdr.index(k)]]

    print(f"# {title}")
    print(f"# {'kernel':22s} {'us':>8s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>7s} {'tensor%':>7s} {'L1%':>6s} {'L2%':>6s} {'DRAMcyc%':>8s}")
    for r in rows[2:]:
        tu = units[hdr.index("gpu__time_duration.sum")]
        t = val(r, "gpu__time_duration.sum") * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                                 "ms": 1e3, "msecond": 1e3}.get(tu, 1.0)
        rd, wr = mb(r, "dram__bytes_read.sum"), mb(r, "dram__bytes_write.sum")
        print(f"{r[hdr.index('Kernel Name')].split('(')[0][:22]:24s} {t:8.1f} {rd:9.1f} {wr:9.1f} {(rd + wr) / t * 1e3:7.0f} "
              f"{val(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):7.1f} "
              f"{val(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{val(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{val(r, 'dram__cycles_active.avg.pct_of_peak_sustained_elapsed'):8.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
