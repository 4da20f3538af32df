"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo + --import-source).

    python tools/ncu_lines.py report.ncu-rep k_force [top]
Prints the lines with the most warp-stall samples and executed instructions, with the
dominant stall reasons (the `--page source --print-source cuda,sass` view, CUDA rows only).
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    rows, hdr, fname = [], None, ""
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or not rec[0] or rec[0] == "Function Name":
            continue
        d = dict(zip(hdr, rec))
        try:
            samp = int(d["Warp Stall Sampling (All Samples)"])
            inst = int(d["Instructions Executed"])
        except (ValueError, KeyError):
            continue
        stalls = {k[6:]: int(v) for k, v in zip(hdr, rec) if k.startswith("stall_") and "Not Issued" not in k
                  and v.isdigit() and int(v) > 0}
        rows.append((samp, inst, f"{fname}:{rec[0]}", rec[1].strip()[:90], stalls))
    ts = sum(r[0] for r in rows) or 1
    ti = sum(r[1] for r in rows) or 1
    print(f"total samples {ts}, warp instructions {ti}")
    for samp, inst, loc, src, stalls in sorted(rows, reverse=True)[:top]:
        st = ", ".join(f"{k} {v}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:3])
        print(f"{100 * samp / ts:5.1f}% smp {100 * inst / ti:5.1f}% ins  {loc:24s} {src}  [{st}]")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
