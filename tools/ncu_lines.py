"""Warp-stall samples per CUDA source line from an ncu report (run here on a
report brought back from the GPU box; needs -lineinfo builds):
    python tools/ncu_lines.py REPORT.ncu-rep [top_n]
Prints the top source lines by 'Warp Stall Sampling (All Samples)' with the
executed-instruction count, and the share of the kernel's samples."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = []
    fname = ""
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0]:
            continue
        try:
            s = int(row[4])
            ex = int(row[7]) if row[7] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        lines.append((s, ex, fname, row[0], row[1].strip()[:90]))
    tot = sum(x[0] for x in lines) or 1
    print("total samples", tot)
    for s, ex, f, ln, src in sorted(lines, reverse=True)[:top]:
        print("%6d %5.1f%% %10d  %s:%s  %s" % (s, 100.0 * s / tot, ex, f, ln, src))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
