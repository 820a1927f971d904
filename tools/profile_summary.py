"""Turn the ncu captures of a round into the committed summaries under profiles/.

    python tools/profile_summary.py <round tag> <capture dir>
e.g. python tools/profile_summary.py r01 gpurun_out/r01

Inputs (made by tools/gpu_prof.sh on the GPU box):
  launches_<workload>.csv  ncu --metrics gpu__time_duration.sum --clock-control none launch lists
  full_<kernel>.ncu-rep    one ncu --set full capture per hot kernel
Outputs:
  profiles/<tag>_launches_<workload>.csv   per-kernel launch count / mean / share of our step
  profiles/<tag>_full_<kernel>.txt          key raw metrics of the --set full capture
  profiles/traffic.json                     dram bytes (read + write) per launch and per voxel,
                                            which bench.py reports as roofline.traffic
"""
import csv
import glob
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(__file__))
from ncu_raw_summary import WANT  # noqa: E402

OURS = re.compile(r"k_step_|k_hist_to_raw|k_mi_finalize|k_zero|k_reduce|k_pad|k_sampler|k_lncc|k_mi_|k_conv|"
                  r"k_add_partials|k_smooth|k_trilinear|k_normalize|k_mse|k_jacobian")
VOXELS = {"mi256": 256 ** 3, "lncc720": 720 * 640 * 720, "wu720": 720 * 640 * 720, "mi1760": 1760 * 1760 * 1200}


def short(name):
    m = re.search(r"(k_[A-Za-z0-9_]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name.split("(")[0][:60]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    agg = OrderedDict()
    for r in rows:
        k = short(r[4])
        ns = float(r[14])
        a = agg.setdefault(k, [0, 0.0, r[7], r[8]])
        a[0] += 1
        a[1] += ns
    ours_total = sum(v[1] for k, v in agg.items() if OURS.search(k))
    with open(out, "w", newline="") as fo:
        w = csv.writer(fo)
        w.writerow(["kernel", "ours", "launches", "mean_us", "total_us", "share_of_our_time", "block", "grid"])
        for k, (n, tot, blk, grd) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            ours = bool(OURS.search(k))
            w.writerow([k, int(ours), n, round(tot / n / 1e3, 3), round(tot / 1e3, 1),
                        round(tot / ours_total, 4) if ours else "", blk, grd])
    return agg


def full(rep, out, workload):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {}
    with open(out, "w") as fo:
        fo.write(f"# ncu --set full --clock-control none capture, workload {workload} ({os.path.basename(rep)})\n")
        for r in rows[2:]:
            name = short(r[ix["Kernel Name"]])
            fo.write(f"== {name}\n")
            for wname in WANT:
                if wname in ix:
                    fo.write(f"   {wname:65s} {r[ix[wname]]:>18s} {units[ix[wname]]}\n")

            def val(key):
                v = float(r[ix[key]].replace(",", ""))
                u = units[ix[key]]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

            stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), float(r[i] or 0)) for i, h in enumerate(hdr)
                if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")),
                key=lambda kv: -kv[1])[:6]
            fo.write("   top warp stall reasons (per issue): " +
                     ", ".join(f"{k} {v:.2f}" for k, v in stalls) + "\n")
            traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            nv = VOXELS[workload]
            fo.write(f"   traffic (dram read + write) per launch: {traffic:.4e} B = {traffic / nv:.2f} B/voxel "
                     f"over {nv} voxels\n")
            key = name.split("<")[0] if workload != "wu720" else name  # the two k_smooth kernels
            res[key] = {"workload": workload, "dram_bytes_per_launch": traffic,
                                       "voxels": nv, "bytes_per_voxel": round(traffic / nv, 3)}
    return res


def main(tag, d):
    os.makedirs("profiles", exist_ok=True)
    for p in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
        wl = os.path.basename(p)[len("launches_"):-4]
        launches(p, f"profiles/{tag}_launches_{wl}.csv")
    traffic = {}
    tp = "profiles/traffic.json"
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for p in sorted(glob.glob(os.path.join(d, "full_*.ncu-rep"))):
        k = os.path.basename(p)[len("full_"):-len(".ncu-rep")]
        # full_<kernel>[_<workload>] or full_<workload>
        wl = next((w for w in VOXELS if w in k), None) or (
            "lncc720" if "lncc" in k else "wu720" if k.startswith("wu") else "mi256")
        for name, v in full(p, f"profiles/{tag}_full_{k}.txt", wl).items():
            v["round"] = tag
            traffic[name] = v
    json.dump(traffic, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
