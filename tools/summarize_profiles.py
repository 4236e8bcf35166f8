"""Turn a profile_round.sh output directory into the committed evidence:

    python tools/summarize_profiles.py gpurun_out/prof3 round1

writes profiles/<tag>_cfg<N>_launches.csv (the raw ncu launch list),
profiles/<tag>_summary.md (per-config launch breakdown + key metrics of the
full captures) and profiles/traffic.json (dram bytes per launch of the
dominant pass kernel, read by bench.py for roofline.traffic).
"""

import csv
import glob
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import summarize  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * UNITS.get(units[i], 1.0)
                except ValueError:
                    pass
                d[m] = v
        res.append(d)
    return res


def main(src, tag):
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lines = [f"# ncu evidence, {tag}", "",
             "Produced by `tools/profile_round.sh` on one B200 (ncu 2025, `--clock-control none`),",
             "summarised by `tools/summarize_profiles.py`. Launch lists cover only the timed",
             "steps of `bench.py` (NVTX range `lr_timed`); ncu serialises launches and runs",
             "cold, so absolute times exceed the bench's CUDA-event times -- the shares are",
             "what must agree. Byte units are bytes, times microseconds.", ""]
    traffic_path = os.path.join(prof, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for lf in sorted(glob.glob(os.path.join(src, "launches_cfg*.csv"))):
        cfg = os.path.basename(lf)[len("launches_"):-4]
        shutil.copy(lf, os.path.join(prof, f"{tag}_{cfg}_launches.csv"))
        bj = os.path.join(src, f"bench_{cfg}.json")
        steps = 2
        if os.path.exists(bj):
            txt = open(bj).read().strip().splitlines()
            if txt:
                b = json.loads(txt[-1])
                steps = int(b.get("steps", 2))
                lines += [f"## {cfg}: {b['config']['workload']}", "",
                          f"bench ({steps} steps, no ncu): {b['ms_per_step']} ms/step, "
                          f"{b['value']} {b['unit']}; roofline kernel frac "
                          f"{b['roofline']['frac']}", ""]
        # the launch lists come from `bench.py --steps 2` (tools/profile_round.sh),
        # whatever step count the bench line beside them was measured with
        lines += ["```", summarize(lf, 2), "```", ""]
        for kind in ("pass", "small"):
            rep = os.path.join(src, f"full_{cfg}_{kind}.ncu-rep")
            if not os.path.exists(rep):
                continue
            shutil.copy(rep, os.path.join(prof, f"{tag}_{cfg}_{kind}.ncu-rep"))
            ms = raw_metrics(rep)
            lines += [f"### `--set full` capture: {kind} kernels ({os.path.basename(rep)})", "",
                      "| kernel | grid | time us | DRAM read B | DRAM write B | SM % | mem % | "
                      "tensor pipe % |", "|---|---|---|---|---|---|---|---|"]
            for d in ms:
                lines.append(
                    f"| {d['kernel'][:60]} | {d.get('launch__grid_size', '')} | "
                    f"{d.get('gpu__time_duration.sum', 0):.1f} | "
                    f"{d.get('dram__bytes_read.sum', 0):.4g} | {d.get('dram__bytes_write.sum', 0):.4g} | "
                    f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                    f"{d.get('gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                    f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} |")
            lines.append("")
            if kind == "pass" and ms:
                # the pass launches proper (a capture may include shorter
                # products of the same kernel, e.g. cfg4's Y P applies)
                tmax = max(d.get("gpu__time_duration.sum", 0) for d in ms)
                big = [d for d in ms if d.get("gpu__time_duration.sum", 0) >= 0.5 * tmax]
                tb = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                      for d in big]
                traffic[cfg] = int(sum(tb) / len(tb))
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    open(os.path.join(prof, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
