"""Summarise an ncu --set full report: key metrics + top stall source lines (for profiles/)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "local_load", "lts__t_bytes.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, kernel_regex=None, top=25):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    out = {}
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")]
        if kernel_regex and kernel_regex not in name:
            continue
        m = {}
        for i, h in enumerate(hdr):
            if any(h == k or (k in h and "pct" not in k and h.startswith(k)) for k in KEYS):
                m[h] = (row[i], units[i])
        out.setdefault(name[:90], m)
    for k, m in out.items():
        print("==", k)
        for h, (v, u) in sorted(m.items()):
            print(f"   {h} = {v} {u}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    # find header row
    hi = next(i for i, r in enumerate(src) if "Warp Stall Sampling (All Samples)" in r)
    h = src[hi]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_src = h.index("Source")
    rows = [r for r in src[hi + 1:] if len(r) > i_s and r[i_s].replace('.', '').isdigit()]
    tot = sum(float(r[i_s]) for r in rows)
    print(f"-- top stall lines ({tot:.0f} samples)")
    for r in sorted(rows, key=lambda r: -float(r[i_s]))[:top]:
        print(f"   {float(r[i_s]) / tot * 100:5.1f}%  {r[0][-6:]}  {r[i_src].strip()[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
