"""Summarize an ncu report: one block per profiled launch with the metrics the roofline
and the design decisions use. Usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("lts__t_sectors_srcunit_tex.sum", "l2_sectors_from_sm"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    # tcgen05 tensor-pipe activity (the sm_100 raw page names it sm__mem_tensor_*; the
    # Hopper-era sm__pipe_tensor_cycles_active* names are absent); any other raw metric
    # mentioning the tensor pipe is listed below the fixed keys
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pct_elapsed"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pct_active"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "xbar2sm_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx.get("Kernel Name", 0)] if "Kernel Name" in idx else "?"
        print(f"--- {name[:80]}")
        for key, label in KEYS:
            if key in idx:
                print(f"  {label:20s} {r[idx[key]]:>16s} {units[idx[key]]}")
        fixed = {k for k, _ in KEYS}
        for h, i in idx.items():
            if (h not in fixed and h.startswith(("sm__pipe_tensor_cycles_active.avg",
                                                  "sm__pipe_tensor_subpipe_hmma"))
                    and r[i] not in ("", "n/a")):
                print(f"  {h[:70]:70s} {r[i]:>10s} {units[i]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"=== {p}")
        main(p)
