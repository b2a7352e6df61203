"""Per-source-line instruction counts and SIMT lane activity from an ncu report
(warp instructions executed, average active threads per instruction).

    python tools/ncu_lanes.py report.ncu-rep [top]
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
    ie, te = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    inst = {r[0]: (float(r[ie] or 0), float(r[te] or 0), r[1]) for r in sass[2:] if len(r) > te}
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
            cur_line = (cur_file, r[0], r[1][:70])
        if len(r) > 2 and r[2].startswith("0x"):
            a2l[r[2]] = cur_line
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    ops = collections.Counter()
    for a, (w, t, src) in inst.items():
        key = a2l.get(a, ("?", "?", "?"))
        agg[key][0] += w
        agg[key][1] += t
        ops[src.split()[0].split(".")[0] if src else "?"] += w
    tot = sum(v[0] for v in agg.values()) or 1
    tt = sum(v[1] for v in agg.values())
    print(f"warp instructions {tot:.3e}, avg active threads {tt / tot:.2f}")
    print("opcode mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(16)))
    for key, (w, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{w / tot * 100:5.1f}%  thr {t / w if w else 0:5.1f}  {key[0]}:{key[1]} {key[2]}")


if __name__ == "__main__":
    main()
