"""Per-launch DRAM traffic and on-chip utilisation of the dominant kernel, from one ncu --set full
capture, into profiles/<round>_traffic.json (read by bench.py: roofline.traffic, roofline.onchip).

    python tools/ncu_traffic.py <capture.ncu-rep> <kernel regex> <config> <level> <launches per level> \
        <voxels per launch> <out.json> [--commit SHA]

The capture is one launch of the level (e.g. the first level-0 slab of config 4, one of 8 launches);
per-level bytes = per-launch bytes x launches per level.
"""
import csv
import io
import json
import re
import subprocess
import sys


def main(argv):
    path, regex, config, level, nlaunch, vox, out = argv[:7]
    commit = argv[argv.index("--commit") + 1] if "--commit" in argv else None
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    row = next(r for r in rows[2:] if re.search(regex, r[hdr.index("Kernel Name")]))

    def num(key):
        v = row[hdr.index(key)].replace(",", "")
        u = units[hdr.index(key)]
        x = float(v)
        return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
                    "ns": 1e-9}.get(u, 1.0)

    per_launch = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    try:
        doc = json.load(open(out))
    except (OSError, ValueError):
        doc = {}
    doc.setdefault(config, {})[level] = {
        "kernel": re.sub(r"[(].*", "", row[hdr.index("Kernel Name")]),
        "bytes_per_launch": per_launch,
        "launches_per_level": int(nlaunch),
        "bytes_per_level": per_launch * int(nlaunch),
        "voxels_per_launch": int(vox),
        "bytes_per_voxel": per_launch / int(vox),
        "ncu_duration_s": num("gpu__time_duration.sum"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "grid_size": int(num("launch__grid_size")),
        "cluster_dim": int(num("launch__cluster_dim_x")),
        "source": path, "commit": commit,
    }
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc[config][level], indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
