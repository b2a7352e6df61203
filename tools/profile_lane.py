"""Write the round-2 profile summaries under profiles/r02/ from a GPU run's raw
outputs (read here, on the build container, with ncu -i):

    python tools/profile_lane.py --lane gpurun_out/lane_full.ncu-rep \
        --launches gpurun_out/launches_r02.csv [--out profiles/r02]

lane: `ncu --set full --clock-control none --import-source on -k regex:lane_kernel
-s 0 -c 1 python tools/profile_step.py --config 3 --queries 50000000 --reps 1`
(one launch over the whole set); launches: `ncu --metrics gpu__time_duration.sum
--clock-control none -c 400 --csv --log-file ... python bench.py --steps 2
--warmup 1 --no-cpu`.  bench.py reads roofline_traffic.json for the `traffic`
and `ncu_counters` of its roofline object.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from profile_summaries import TO_BASE, kernel_summary, launches, num  # noqa: E402

LANE_CMD = ("ncu --set full --clock-control none --import-source on -k regex:lane_kernel -s 0 -c 1 "
            "python tools/profile_step.py --config 3 --queries 50000000 --reps 1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lane", required=True)
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "r02"))
    args = ap.parse_args()
    out = args.out
    det, raw = kernel_summary(args.lane)
    lanes_txt = subprocess.run([sys.executable, os.path.join(HERE, "ncu_lanes.py"), args.lane, "30"],
                               capture_output=True, text=True, check=True).stdout
    stalls = subprocess.run([sys.executable, os.path.join(HERE, "ncu_lines.py"), args.lane, "30"],
                            capture_output=True, text=True, check=True).stdout
    lines = ["# ncu --set full, lane_kernel, full config 3 (5e7 queries, one launch), B200",
             f"# command: {LANE_CMD}"]
    lines += [f"{k}: {v} {u}".rstrip() for k, (v, u) in det.items()]
    lines += [f"{k} | {v} {u}".rstrip() for k, (v, u) in raw.items()]
    lines += ["", "# instruction mix and per-line SIMT activity (tools/ncu_lanes.py)", lanes_txt.rstrip(),
              "", "# warp stall samples per source line (tools/ncu_lines.py)", stalls.rstrip()]
    with open(os.path.join(out, "lane_ncu_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")

    val = lambda k: num(raw[k][0]) * TO_BASE.get(raw[k][1], 1.0)  # noqa: E731
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur_s = val("gpu__time_duration.sum")
    act = num(raw["smsp__thread_inst_executed_per_inst_executed.ratio"][0])
    t = {"kernel": "lane", "config": 3, "queries": 50000000,
         "dram_bytes_per_launch": int(rd + wr), "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
         "source": LANE_CMD + " (one launch over the whole set); summary in lane_ncu_summary.txt",
         "note": "DRAM traffic per launch against ~9.6 GB of algorithmic input traffic for the whole step "
                 "(the lane kernel re-reads the coordinates of its 2.7e7 queries, 5.2 GB, plus 64-B records "
                 "1.7 GB, plus its level entries): a few percent of HBM peak, not memory-bound",
         "fp64_pipe_active_pct": round(num(raw["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]), 2),
         "warp_execution_efficiency_pct": round(act / 32 * 100, 1),
         "avg_active_threads_per_warp": act,
         "dram_gbs": round((rd + wr) / dur_s / 1e9, 1),
         "issue_slots_busy_pct": num(det["Issue Slots Busy"][0]),
         "duration_ms_under_ncu": round(dur_s * 1e3, 2),
         "l2_hit_pct": round(num(raw["lts__t_sector_hit_rate.pct"][0]), 2)}
    with open(os.path.join(out, "roofline_traffic.json"), "w") as fh:
        json.dump(t, fh, indent=1)
    print(json.dumps(t))

    if args.launches:
        agg = launches(args.launches)
        with open(args.launches) as src, open(os.path.join(out, "launches_r02.csv"), "w") as dst:
            dst.write(src.read())
        tot = sum(a[1] for a in agg.values())
        md = ["# Launch list of `python bench.py --steps 2 --warmup 1 --no-cpu` (config 3, 5e7 queries)", "",
              "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv` (cold-cache, serialized: "
              "compare shares, not absolutes).  The run solves the set several times (one untimed full-output "
              "solve, the warm-up, the timed device steps, the e2e warm-up and steps); engine kernels launch "
              "once per sub-chunk of the light queue (most of them on an empty slice).", "",
              "| kernel | launches | total ms | share of tccd time | ms per launch |", "|---|---|---|---|---|"]
        for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{k[:70]}` | {n} | {ms:.2f} | {100 * ms / tot:.1f}% | {ms / n:.3f} |")
        with open(os.path.join(out, "launches_summary.md"), "w") as fh:
            fh.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
