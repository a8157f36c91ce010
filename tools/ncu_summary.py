"""Condense an ncu report (--set full) into the numbers DESIGN.md / profiles/ cite.

    python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]

Prints: duration, clocks, issue/pipe utilisation (FMA, ALU, XU = MUFU, LSU),
DRAM bytes per launch, shared-memory wavefronts and bank conflicts, occupancy,
warp-stall breakdown, and the SASS instruction mix (with FFMA2 counted as two
FP32 lanes per thread).
"""
import collections
import csv
import io
import json
import subprocess
import sys


def _csv(args):
    out = subprocess.run(["ncu", "-i"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = _csv([rep, "--page", "raw"])
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({name: (unit, val) for name, unit, val in zip(h, u, v)})
    return res


def num(m, k, default=None):
    try:
        return float(m[k][1].replace(",", ""))
    except (KeyError, ValueError):
        return default


def sass_mix(rep):
    rows = _csv([rep, "--page", "source", "--print-source", "sass"])
    if len(rows) < 3:
        return {}
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    mix = collections.Counter()
    stall = collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        try:
            mix[op] += int(r[ix["Instructions Executed"]] or 0)
            stall[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            pass
    return {"mix": dict(mix.most_common(25)), "stall_samples": dict(stall.most_common(12))}


def summarize(rep):
    out = []
    for m in raw_metrics(rep):
        name = m.get("Kernel Name", ("", ""))[1]
        dur = num(m, "gpu__time_duration.sum")
        s = {
            "kernel": name[:120],
            "duration_ms": dur,
            "sm_mhz": (num(m, "sm__cycles_elapsed.avg.per_second") or 0) * {"Ghz": 1e3, "GHz": 1e3, "Mhz": 1.0, "MHz": 1.0, "hz": 1e-6}.get(m.get("sm__cycles_elapsed.avg.per_second", ("", ""))[0], 1.0),
            "regs": num(m, "launch__registers_per_thread"),
            "smem_per_block_kb": (num(m, "launch__shared_mem_per_block_dynamic") or 0) *
                                 {"byte": 1 / 1024, "Kbyte": 1000 / 1024, "Mbyte": 1e6 / 1024}.get(
                                     m.get("launch__shared_mem_per_block_dynamic", ("", ""))[0], 1),
            "achieved_occupancy_pct": num(m, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num(m, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "inst_executed": num(m, "smsp__inst_executed.sum"),
            "pipe_fma_pct": num(m, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "pipe_fma_cycles_pct": num(m, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "pipe_alu_pct": num(m, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "pipe_xu_pct": num(m, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "pipe_lsu_pct": num(m, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "dram_read_bytes": num(m, "dram__bytes_read.sum"),
            "dram_write_bytes": num(m, "dram__bytes_write.sum"),
            "smem_wavefronts": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_bank_conflicts": num(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "smem_wavefront_pct": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        }
        stalls = {}
        for k in m:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                v = num(m, k)
                if v and v > 0.01:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        # unit fixups: dram bytes reported in the unit column
        for key, mk in (("dram_read_bytes", "dram__bytes_read.sum"), ("dram_write_bytes", "dram__bytes_write.sum")):
            unit = m.get(mk, ("", ""))[0]
            if s[key] is not None:
                s[key] *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        dur_unit = m.get("gpu__time_duration.sum", ("", ""))[0]
        if dur is not None:
            s["duration_ms"] = dur * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(dur_unit, 1e-6)
        out.append(s)
    mix = sass_mix(rep)
    return {"launches": out, "sass": mix}


if __name__ == "__main__":
    rep = sys.argv[1]
    res = summarize(rep)
    txt = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt)
    print(txt)
