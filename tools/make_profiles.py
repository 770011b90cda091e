"""Summarise this round's ncu captures into profiles/ (tracked): per-kernel text summaries,
the launch-list shares of the bench command, and profiles/ncu_summary.json (read by bench.py).

    python tools/make_profiles.py TAG     # reads gpurun_out/*_TAG.*
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

# (capture name, kernel key used by bench.py, algorithmic bytes per launch, description)
CAPTURES = [
    ("cfg2_prefill", "prefill_tc", 8 * 32 * 8192 * 1024, "configs[1] B=8,H=32,N=8192,d=128: one launch, no split"),
    ("cfg3_prefill", "prefill_tc_dk256", 4 * 16 * 16384 * 3072, "configs[2] B=4,H=16,N=16384,dk=256,dv=512"),
    ("cfg5_statepass", "state_pass_split", 32 * 98304 * 512, "configs[4] phase A: K,V of segments 0..2 (98304 tokens x 32 heads)"),
    ("cfg5_prefill", "prefill_split", 32 * 131072 * 1024, "configs[4] phase B: 4 seeded segments x 32 heads"),
    ("decode", "decode_step", 256 * 32 * 132096, "configs[3] decode step B=256,H=32,d=128"),
    ("fp32_prefill", "prefill_simt_fp32", 8 * 32 * 2048 * 2048,
     "fp32 FFMA kernel B=8,H=32,N=2048,d=128 (tools/f32_once.py): balanced, cp.async staging"),
    ("tf32_prefill", "prefill_tf32", 8 * 32 * 8192 * 2048,
     "fp32 parity mode on the tensor cores (3xTF32) at the configs[1] shape B=8,H=32,N=8192,d=128"),
]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for k in METRICS:
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1e3, "us": 1, "ns": 1e-3}.get(units[i], 1)
            try:
                m[k] = float(v) * scale
            except ValueError:
                m[k] = v
    m["kernel"] = vals[hdr.index("Kernel Name")][:100]
    return m


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            tot[r[ik]][0] += 1
            tot[r[ik]][1] += float(r[iv].replace(",", "")) / 1e3   # ns -> us
    allt = sum(v[1] for v in tot.values())
    lines = []
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{n:6d} launches  mean {t / n:10.1f} us  total {t:10.1f} us  share {100 * t / allt:5.1f}%  {k[:110]}")
    return lines


def main(tag):
    gout = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    rnd = tag[:2] if tag[:1] == "r" and tag[1:2].isdigit() else "r"
    summary = {"_source": f"ncu --set full --clock-control none, one launch per kernel (round tag {tag}); "
                          f"per-kernel summaries in profiles/{rnd}_<name>_ncu.txt"}
    import ncu_summary
    for name, key, alg, desc in CAPTURES:
        rep = os.path.join(gout, f"prof_{name}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m = raw_metrics(rep)
        t_us = m.get("gpu__time_duration.sum", 0.0)
        traffic = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        summary[key] = {"workload": desc, "kernel": m["kernel"], "gpu_time_us_ncu": t_us,
                        "dram_read": m.get("dram__bytes_read.sum"), "dram_write": m.get("dram__bytes_write.sum"),
                        "dram_bytes_per_launch": traffic, "algorithmic_bytes_per_launch": alg,
                        "traffic_over_algorithmic": traffic / alg if alg else None,
                        "algorithmic_GBps_ncu": alg / (t_us * 1e-6) / 1e9 if t_us else None,
                        "tensor_pipe_active_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                        "dram_throughput_pct": m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                        "grid": m.get("launch__grid_size"), "block": m.get("launch__block_size"),
                        "registers": m.get("launch__registers_per_thread"),
                        "smem_tc_wavefronts_pct": m.get(
                            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                        "smem_lsu_wavefronts_pct": m.get(
                            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")}
        buf = io.StringIO()
        old = sys.stdout
        sys.stdout = buf
        try:
            ncu_summary.main(rep, None, 30)
        finally:
            sys.stdout = old
        with open(os.path.join(prof, f"{rnd}_{name}_ncu.txt"), "w") as fh:
            fh.write(f"# {desc}\n# ncu --set full --clock-control none --import-source on (tools/gpu_profile.sh {tag})\n")
            fh.write(buf.getvalue())
    with open(os.path.join(prof, "ncu_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    lpath = os.path.join(gout, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        with open(os.path.join(prof, f"{rnd}_launches_summary.txt"), "w") as fh:
            fh.write("ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 3 --warmup 3 "
                     "--no-cpu --decode-steps 64\n(cold-cache, serialised per-launch times; compare shares, not "
                     "absolutes)\n")
            fh.write("\n".join(launch_shares(lpath)) + "\n")
        subprocess.run(["cp", lpath, os.path.join(prof, f"{rnd}_launches.csv")])


if __name__ == "__main__":
    main(sys.argv[1])
