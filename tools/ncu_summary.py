"""Summarise an ncu report: one line per kernel launch with the metrics that
matter for an HBM-bound kernel."""
import csv
import io
import subprocess
import sys

WANT = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sect"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    cols = [(hdr.index(k), n) for k, n in WANT if k in hdr]
    print(" | ".join(f"{n}[{units[i]}]" if units[i] else n for i, n in cols))
    for r in rows[2:]:
        print(" | ".join(r[i][:34] for i, _ in cols))


if __name__ == "__main__":
    main(sys.argv[1])
