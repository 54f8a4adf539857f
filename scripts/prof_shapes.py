"""Per-launch-shape ncu counters for bench.py's rooflines (dev/profiling aid;
run on the GPU box).  For every bench line it captures the DAS launches of
ONE beamform call with

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
                dram__bytes_write.sum,smsp__inst_executed.sum,
                lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct

and writes profiles/das_ncu.json entries {frames, dram_bytes_per_launch,
warp_inst_per_launch, l2_hit_rate, l1_hit_rate, ...} summed over the call's DAS launches (main +
remainder).  ncu replays each kernel, so times here are cold-cache and
serialised: only the counters are used.

  python scripts/prof_shapes.py [KEY ...]     # default: all bench shapes
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# key -> (config, frames per call, DAS launches per call)
SHAPES = {
    "C2": ("C2", 100, 2), "C3": ("C3", 32, 1), "C4a": ("C4a", 1, 1), "C4a_stream": ("C4a", 2, 1), "C4b": ("C4b", 8, 1),
    "C4b_1": ("C4b", 1, 1), "C4p": ("C4p", 4, 1), "C4p_1": ("C4p", 1, 1),
    "T1_64_1": ("T1_64_1", 64, 1), "T1_64_2": ("T1_64_2", 64, 1),
    "T1_128_1": ("T1_128_1", 64, 1), "T1_128_2": ("T1_128_2", 64, 1),
}
METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,"
           "lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct")


def capture(cfg, F, nl, reps=3):
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--print-units", "base", "-k", "regex:das_",
           "-s", str((reps - 1) * nl), "-c", str(nl), sys.executable,
           os.path.join(ROOT, "scripts", "prof_das.py"), cfg, str(F), str(reps)]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):]))] if '"ID"' in out else []
    hdr, body = rows[0], rows[1:]
    i_name, i_met, i_val = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    i_id = hdr.index("ID")
    per = {}
    for r in body:
        per.setdefault(r[i_id], {"kernel": r[i_name]})[r[i_met]] = float(r[i_val].replace(",", ""))
    return list(per.values())


def main():
    keys = sys.argv[1:] or list(SHAPES)
    path = os.path.join(ROOT, "profiles", "das_ncu.json")
    try:
        db = json.load(open(path))
    except (OSError, ValueError):
        db = {}
    db["_doc"] = ("Per bench line: counters of the DAS launches of ONE beamform call (main + remainder "
                  "launch), from ncu --metrics " + METRICS + " (scripts/prof_shapes.py); read by bench.py "
                  "as roofline.traffic (DRAM read + write) and the ALU roofline's warp instructions.")
    for k in keys:
        cfg, F, nl = SHAPES[k]
        launches = capture(cfg, F, nl)
        if len(launches) != nl:
            print(k, "capture failed", launches, flush=True)
            continue
        e = {"config": cfg, "frames": F, "launches": [l["kernel"][:80] for l in launches],
             "dram_read": sum(l["dram__bytes_read.sum"] for l in launches),
             "dram_write": sum(l["dram__bytes_write.sum"] for l in launches),
             "warp_inst_per_launch": sum(l["smsp__inst_executed.sum"] for l in launches),
             "ncu_time_ms": sum(l["gpu__time_duration.sum"] for l in launches) / 1e6}
        # hit rates of the call's launches, weighted by their (ncu) time
        tw = sum(l["gpu__time_duration.sum"] for l in launches)
        for m, key in (("lts__t_sector_hit_rate.pct", "l2_hit_rate"), ("l1tex__t_sector_hit_rate.pct", "l1_hit_rate")):
            if all(m in l for l in launches):
                e[key] = sum(l[m] * l["gpu__time_duration.sum"] for l in launches) / tw / 100.0
        e["dram_bytes_per_launch"] = e["dram_read"] + e["dram_write"]
        db[k] = e
        print(k, json.dumps(e), flush=True)
        json.dump(db, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
