"""Aggregate ncu warp-stall samples per CUDA source line.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", *args],
                          capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    sass = list(csv.reader(io.StringIO(run(rep, "--print-source", "sass"))))
    mix = list(csv.reader(io.StringIO(run(rep, "--print-source", "cuda,sass"))))
    h = sass[1]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    samp = {r[0]: float(r[i_s] or 0) for r in sass[2:] if len(r) > i_s}
    reasons = [(k, c) for k, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    why = {r[0]: {c: float(r[k] or 0) for k, c in reasons} for r in sass[2:] if len(r) > i_s}
    cur_file, cur_line, a2l = None, None, {}
    for r in mix:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0].startswith("=="):
            continue
        if r[0] != "":
            cur_line = (cur_file, r[0], r[1][:80])
        if len(r) > 2 and r[2].startswith("0x"):
            a2l[r[2]] = cur_line
    agg = collections.Counter()
    agg_why = collections.defaultdict(collections.Counter)
    overall = collections.Counter()
    for a, s in samp.items():
        key = a2l.get(a, ("?", "?", "?"))
        agg[key] += s
        agg_why[key].update(why[a])
        overall.update(why[a])
    tot = sum(samp.values()) or 1
    print("stall reasons:", ", ".join(f"{c[6:]} {v / tot * 100:.1f}%"
                                      for c, v in overall.most_common(8)))
    for k, v in agg.most_common(top):
        top3 = ", ".join(f"{c[6:]} {x / v * 100:.0f}%" for c, x in agg_why[k].most_common(3) if v)
        print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]} {k[2][:60]}  [{top3}]")


if __name__ == "__main__":
    main()
