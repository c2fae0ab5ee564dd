"""Summarise ncu evidence into profiles/ (committed; gpurun_out/ is scratch).

  python tools/ncu_summary.py kernel <prof_tag> <out.txt> [algorithmic_bytes_per_launch]
      one `ncu --set full` capture (raw + sass csv from tools/prof_kernel.sh)
  python tools/ncu_summary.py launches <launches.csv> <out.txt> <steps_in_capture> [decode_scale]
      the `--metrics gpu__time_duration.sum` launch list of a bench run
"""
import collections
import csv
import io
import subprocess
import sys

RAW_KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "HMMA pipe active %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def _to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    return None if f is None else float(v) * f


def kernel(tag, out, alg_bytes=None):
    rows = list(csv.reader(open(f"gpurun_out/prof_{tag}.raw.csv")))
    hdr, units, val = rows[0], rows[1], rows[2]
    lines = [f"ncu --set full --clock-control none capture '{tag}' (one launch, cold caches, serialised)",
             f"kernel: {val[hdr.index('Kernel Name')]}", ""]
    got = {}
    for key, label in RAW_KEYS:
        if key in hdr:
            i = hdr.index(key)
            got[key] = (val[i], units[i])
            lines.append(f"  {label:32s} {val[i]:>14s} {units[i]}  [{key}]")
    rd = _to_bytes(*got["dram__bytes_read.sum"])
    wr = _to_bytes(*got["dram__bytes_write.sum"])
    us = float(got["gpu__time_duration.sum"][0]) * {"usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}[
        got["gpu__time_duration.sum"][1]]
    lines.append("")
    lines.append(f"  traffic (read+write)              {rd + wr:.0f} bytes/launch")
    lines.append(f"  DRAM GB/s under ncu               {(rd + wr) / us / 1e3:.1f}")
    if alg_bytes:
        lines.append(f"  algorithmic bytes/launch          {alg_bytes:.0f}  (traffic/algorithmic = {(rd + wr) / alg_bytes:.3f})")
    sass = f"gpurun_out/prof_{tag}.sass.csv"
    try:
        res = subprocess.run([sys.executable, "tools/ana_sass.py", sass, "6"], capture_output=True, text=True)
        lines += ["", "warp-state samples (tools/ana_sass.py over the SASS source page):", res.stdout]
    except Exception as e:   # pragma: no cover
        lines.append(f"(no sass page: {e})")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out, steps, gen_scale=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[r[iu]]
        t[name] += v
        n[name] += 1
    ours = {k: v for k, v in t.items() if k.startswith("wq::")}
    tot = sum(ours.values())
    buf = io.StringIO()
    buf.write(f"ncu --metrics gpu__time_duration.sum --clock-control none launch list of `{path}`\n")
    buf.write(f"libwq kernels only (torch kernels in the list are synthetic-input generation outside the timed region).\n")
    buf.write(f"The capture holds {steps} passes of the step; per-launch times are cold-cache and serialised, so\n")
    buf.write("compare the SHARE of the step, not the absolute time.\n\n")
    buf.write(f"{'kernel':34s} {'launches':>8s} {'avg us':>9s} {'total us':>11s} {'share':>7s}\n")
    for k, v in sorted(ours.items(), key=lambda x: -x[1]):
        buf.write(f"{k[:34]:34s} {n[k]:8d} {v / n[k]:9.2f} {v:11.1f} {100 * v / tot:6.1f}%\n")
    buf.write(f"{'total':34s} {sum(n[k] for k in ours):8d} {'':9s} {tot:11.1f}\n")
    if gen_scale:
        # the capture ran n_gen tokens per step; bench.py's step runs gen_scale x more decode launches
        proj = {k: v * (gen_scale if "k_decode" in k else 1) for k, v in ours.items()}
        pt = sum(proj.values())
        buf.write(f"\nprojected share of bench.py's step (decode launches x{gen_scale}, same per-launch times):\n")
        for k, v in sorted(proj.items(), key=lambda x: -x[1]):
            buf.write(f"{k[:34]:34s} {100 * v / pt:6.1f}%\n")
    open(out, "w").write(buf.getvalue())
    print(buf.getvalue())


if __name__ == "__main__":
    if sys.argv[1] == "kernel":
        kernel(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3], int(sys.argv[4]), float(sys.argv[5]) if len(sys.argv) > 5 else None)
