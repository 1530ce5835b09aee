"""Per-source-line instruction / stall summary of one kernel in an ncu report
(`ncu -i REP --page source --csv --print-source cuda,sass`).

    python profiles/srcprof.py REP KERNEL_REGEX [top] [samp]   (samp: order by stall samples)
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    fname, lines, tot_i, tot_s = None, {}, 0, 0
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row)}
            continue
        if hdr is None or row[0] in ("", "Function Name", "Kernel Name"):
            continue
        try:
            n_inst = int(row[hdr["Instructions Executed"]] or 0)
            samp = int(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            continue
        key = (fname, int(row[0]))
        src = row[1].strip()[:90]
        a = lines.setdefault(key, [0, 0, src])
        a[0] += n_inst
        a[1] += samp
        tot_i += n_inst
        tot_s += samp
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    col = 1 if len(sys.argv) > 4 and sys.argv[4] == "samp" else 0
    for (f, ln), (ni, ss, src) in sorted(lines.items(), key=lambda kv: -kv[1][col])[:top]:
        print(f"{100 * ni / tot_i:5.1f}% inst {100 * ss / max(tot_s, 1):5.1f}% samp  {f}:{ln:<4} {src}")


if __name__ == "__main__":
    main()
