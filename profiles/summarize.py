"""Summarise ncu outputs into small committed files under profiles/.

  python profiles/summarize.py launches <launches.csv> <out.json>
  python profiles/summarize.py full <report.ncu-rep> <out.json> [algorithmic_bytes_per_launch] [iterations_per_launch]
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, order = {}, []
    for r in rows[start + 1:]:
        if len(r) <= ival:
            continue
        name = r[iname].split("(")[0]
        ms = float(r[ival].replace(",", "")) * UNIT.get(r[iunit], 1e-6)
        if name not in agg:
            agg[name] = [0, 0.0]
            order.append(name)
        agg[name][0] += 1
        agg[name][1] += ms
    total = sum(v[1] for v in agg.values())
    res = [{"kernel": k, "launches": agg[k][0], "total_ms": round(agg[k][1], 4),
            "share": round(agg[k][1] / total, 4)} for k in sorted(agg, key=lambda k: -agg[k][1])]
    json.dump({"source": path, "total_ms": round(total, 3), "kernels": res}, open(out, "w"), indent=1)
    for x in res[:12]:
        print(f"{x['launches']:5d} {x['total_ms']:12.3f} ms {100 * x['share']:6.2f}%  {x['kernel']}")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_no_instructions",
        "smsp__pcsamp_warps_issue_stalled_barrier"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full(rep, out, alg=None, iters=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0] if "Kernel Name" in hdr else "?"}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if units[i] in SCALE:
                    v *= SCALE[units[i]]
                    d[w] = v
                else:
                    d[w] = v if units[i] != "nsecond" else v
                    if units[i]:
                        d[w + ".unit"] = units[i]
        if "dram__bytes_read.sum" in d:
            d["dram_bytes_per_launch"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
        if alg:
            d["algorithmic_bytes_per_launch"] = float(alg)
        if iters and "dram_bytes_per_launch" in d:
            d["iterations_per_launch"] = int(iters)
            d["dram_bytes_per_iteration"] = d["dram_bytes_per_launch"] / int(iters)
        kernels.append(d)
    json.dump({"source": rep, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None,
             sys.argv[5] if len(sys.argv) > 5 else None)
