"""Top warp-stall sites of an ncu report (source page, SASS), with the CUDA source line
when -lineinfo is present. Usage: python scripts/ncu_stalls.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass,cuda"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
    hdr = rows[hdr_i]
    data = rows[hdr_i + 1:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    seen, tot = set(), 0
    uniq = []
    for r in data:
        if len(r) <= i_s or not r[i_s].isdigit():
            continue
        key = r[0]
        if key in seen:
            continue
        seen.add(key)
        tot += int(r[i_s])
        uniq.append(r)
    print(f"total samples {tot}")
    for r in sorted(uniq, key=lambda r: -int(r[i_s]))[:n]:
        print(f"{int(r[i_s]) / max(tot, 1):6.1%} {r[i_ex]:>10s} {r[0][-6:]} {r[i_src][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
