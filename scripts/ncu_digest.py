"""Per-kernel digest of an `ncu --page raw --csv` export: duration, DRAM bytes
(read / write / per amplitude for a given N), DRAM throughput %.
Usage: python scripts/ncu_digest.py raw.csv N"""
import csv
import sys


def main(path, N):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                   "dram__bytes_write.sum",
                                   "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
    for r in rows[2:]:  # row 1 holds the units
        if len(r) < len(h) or not r[col["Kernel Name"]]:
            continue
        units = rows[1]
        def val(k):
            v = float(r[col[k]].replace(",", ""))
            u = units[col[k]]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6,
                     "usecond": 1e-3, "msecond": 1.0, "%": 1}.get(u, 1)
            return v * scale
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        print(f'{r[col["Kernel Name"]][:40]:40s} {val("gpu__time_duration.sum"):9.3f} ms  '
              f"read {rd / 1e9:7.2f} GB  write {wr / 1e9:7.2f} GB  {(rd + wr) / N:6.2f} B/amp  "
              f'DRAM {val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):.1f}%')


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
