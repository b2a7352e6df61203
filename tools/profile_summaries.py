"""Write the committed profile summaries under profiles/<round>/ from a GPU run's
raw outputs (read here, on the build container, with ncu -i):

    python tools/profile_summaries.py --bench gpurun_out/bench.log \
        --launches gpurun_out/launches.csv --light gpurun_out/light.ncu-rep \
        --medium gpurun_out/medium.ncu-rep [--out profiles/r01]

bench.log: `python bench.py` output (its JSON line becomes bench_rNN.json);
launches.csv: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400
--csv --log-file ... python bench.py --steps 2 --warmup 3 --no-cpu`;
light / medium: `ncu --set full --import-source on --clock-control none
--kernel-name-base demangled -k regex:3840 (16384) --launch-skip 1 -c 1
python tools/profile_step.py --config 1 --reps 2`.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DETAILS = ["DRAM Throughput", "Duration", "Compute (SM) Throughput", "Executed Ipc Active",
           "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible",
           "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
           "Registers Per Thread", "Theoretical Occupancy", "Achieved Active Warps Per SM"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]
TO_BASE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
           "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


def kernel_summary(rep):
    """(details {name: (value, unit)}, raw {metric: (value, unit)})"""
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    det = {}
    for r in rows[1:]:
        if r[iN] in DETAILS and r[iN] not in det:
            det[r[iN]] = (r[iV], r[iU])
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv", "--metrics", ",".join(RAW)))))
    raw = {n: (rows[2][i], rows[1][i]) for i, n in enumerate(rows[0]) if n in RAW}
    return det, raw


def num(v):
    return float(str(v).replace(",", ""))


def write_kernel(out, name, regex, rep):
    det, raw = kernel_summary(rep)
    lines = [f"# {name} tier (config 1, 10^6 queries, second solve): ncu --set full --import-source on "
             f"--clock-control none --kernel-name-base demangled -k regex:{regex} --launch-skip 1 -c 1 "
             "python tools/profile_step.py --config 1 --reps 2"]
    lines += [f"{k} {v}" for k, (v, _) in det.items()]
    lines += [f"{k} | {v} {u}".rstrip() for k, (v, u) in raw.items()]
    with open(os.path.join(out, f"{name}_tier_ncu_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    stalls = subprocess.run([sys.executable, os.path.join(HERE, "ncu_lines.py"), rep, "30"],
                            capture_output=True, text=True, check=True).stdout
    with open(os.path.join(out, f"{name}_tier_stall_lines.txt"), "w") as fh:
        fh.write(stalls)
    return det, raw


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(r for r in rows if "Kernel Name" in r)
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[rows.index(h) + 1:]:
        if len(r) <= iV or "tccd" not in r[iN]:
            continue
        ms = num(r[iV]) * TO_BASE.get(r[iU], 1e-9) * 1e3
        a = agg.setdefault(r[iN], [0, 0.0])
        a[0] += 1
        a[1] += ms
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--light", required=True)
    ap.add_argument("--medium", default=None)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r01"))
    ap.add_argument("--tag", default="r01")
    args = ap.parse_args()
    out = args.out
    line = next(l for l in open(args.bench) if l.startswith("{"))
    bench = json.loads(line)
    with open(os.path.join(out, f"bench_{args.tag}.json"), "w") as fh:
        fh.write(line if line.endswith("\n") else line + "\n")

    agg = launches(args.launches)
    with open(args.launches) as src, open(os.path.join(out, f"launches_{args.tag}.csv"), "w") as dst:
        dst.write(src.read())
    tot = sum(a[1] for a in agg.values())
    st, ms = bench["roofline"]["stage_ms"], bench["ms_per_step"]
    md = ["# Launch list summary (ncu gpu__time_duration.sum, --clock-control none; cold/serialised)", "",
          "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py "
          "--steps 2 --warmup 3 --no-cpu` (config 1, 10^6 queries; every solve of the run incl. warm-up and e2e)",
          "", "| kernel | launches | total ms | ms / launch | share of tccd time |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        md.append(f"| {k} | {n} | {t:.2f} | {t / n:.3f} | {100 * t / tot:.1f}% |")
    md += ["", f"Bench's own stage split (CUDA events in the timed region, profiles/{args.tag}/bench_{args.tag}.json): "
           f"prologue {st['prologue']:.2f} / light {st['light']:.1f} / medium {st['medium']:.1f} / giant "
           f"{st['giant']:.1f} ms of {ms:.1f} ms -> light {100 * st['light'] / ms:.1f}%, medium "
           f"{100 * st['medium'] / ms:.1f}%, giant {100 * st['giant'] / ms:.1f}% (the giant stage includes the "
           "giant-queue order kernel): compare with the cold serialised shares above."]
    with open(os.path.join(out, "launches_summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")

    det, raw = write_kernel(out, "light", 3840, args.light)
    if args.medium:
        write_kernel(out, "medium", 16384, args.medium)
    val = lambda k: num(raw[k][0]) * TO_BASE.get(raw[k][1], 1.0)  # noqa: E731
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur_s = val("gpu__time_duration.sum")
    tpath = os.path.join(out, "roofline_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lanes = num(raw["smsp__thread_inst_executed_per_inst_executed.ratio"][0])
    t.update({"kernel": "light", "config": 1, "queries": 1000000,
              "dram_bytes_per_launch": int(rd + wr), "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
              "fp64_pipe_active_pct": round(num(raw["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]), 2),
              "warp_execution_efficiency_pct": round(lanes / 32 * 100, 1),
              "avg_active_threads_per_warp": lanes,
              "dram_gbs": round((rd + wr) / dur_s / 1e9, 1),
              "issue_slots_busy_pct": num(det["Issue Slots Busy"][0]),
              "l2_hit_pct": round(num(raw["lts__t_sector_hit_rate.pct"][0]), 2),
              "duration_ms_under_ncu": round(dur_s * 1e3, 3)})
    with open(tpath, "w") as fh:
        json.dump(t, fh, indent=1)
    print(json.dumps({k: t[k] for k in ("dram_bytes_per_launch", "fp64_pipe_active_pct", "dram_gbs",
                                         "issue_slots_busy_pct", "l2_hit_pct", "duration_ms_under_ncu")}))


if __name__ == "__main__":
    main()
