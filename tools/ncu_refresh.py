"""Turn the reports of tools/ncu_capture.sh into profiles/ncu_summary.json entries
and per-kernel briefs.

    python tools/ncu_refresh.py <tag> <round-label>     (reads gpurun_out/<tag>_*)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")
FP64 = {k: f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum" for k in ("dadd", "dmul", "dfma")}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def num(x):
    return float(str(x).replace(",", ""))


def generator(rep, samples, label):
    v, u = raw(rep)
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = num(v["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = num(v["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    t = num(v["gpu__time_duration.sum"]) * {"us": 1e-6, "ns": 1e-9, "ms": 1e-3}[u["gpu__time_duration.sum"]]
    wi = num(v["smsp__inst_executed.sum"])
    ld = num(v["smsp__sass_inst_executed_op_shared_ld.sum"])
    return {
        "kernel": v["Kernel Name"], "duration_s": t, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr, "dram_gbs": (rd + wr) / t / 1e9,
        "registers": num(v["launch__registers_per_thread"]), "grid": num(v["launch__grid_size"]),
        "issue_active_pct": num(v["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "alu_pipe_pct": num(v["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]),
        "fma_pipe_pct": num(v["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]),
        "l1_data_pipe_lsu_wavefronts_pct": num(v["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]),
        "shared_ld_wavefronts": num(v["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]),
        "shared_ld_instructions": ld,
        "shared_wavefronts_per_ld": num(v["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]) / ld if ld else None,
        "samples_per_launch": samples, "warp_instructions": wi,
        "thread_instructions_per_sample": wi * 32 / samples,
        "source": f"gpurun_out/{os.path.basename(rep)} (ncu --set full --clock-control none, {label}; ncu serialises "
                  "and runs a cold single launch: compare shares, not absolute times)",
    }


def gbm(rep, path_steps, label, kernel_note):
    v, u = raw(rep)
    t = num(v["gpu__time_duration.sum"]) * {"us": 1e-6, "ns": 1e-9, "ms": 1e-3}[u["gpu__time_duration.sum"]]
    c = {k: num(v[m]) for k, m in FP64.items()}
    wi = num(v["smsp__inst_executed.sum"])
    return {
        "kernel": kernel_note + " [" + v["Kernel Name"][:60] + "]", "duration_s": t, **c, "path_steps": path_steps,
        "fp64_pipe_active_pct": num(v["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
        "issue_active_pct": num(v["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
        "warps_active_pct": num(v["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "registers": num(v["launch__registers_per_thread"]),
        "active_lanes_per_warp_inst": num(v["smsp__thread_inst_executed_per_inst_executed.ratio"]),
        "dp_flops_per_path_step": (c["dadd"] + c["dmul"] + 2 * c["dfma"]) / path_steps,
        "dp_lane_ops_per_path_step": (c["dadd"] + c["dmul"] + c["dfma"]) / path_steps,
        "warp_instructions_per_32_path_steps": wi * 32 / path_steps,
        "source": f"gpurun_out/{os.path.basename(rep)}, {label}",
    }


def cir(csv_path, path_steps, label, kernel_note):
    """All kernels of one CIR exact level (the last prof_kernels repetition)."""
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 14 and r[0].isdigit()]
    per = collections.defaultdict(dict)
    for r in rows:
        per[int(r[0])][r[12]] = (num(r[14]), r[13], r[4])
    ids = sorted(per)
    half = ids[len(ids) // 2:]  # second repetition (first = warm-up)
    tot = collections.Counter()
    w = collections.Counter()
    for i in half:
        m = per[i]
        t = m["gpu__time_duration.sum"][0] * 1e-9
        tot["t"] += t
        for k, name in FP64.items():
            tot[k] += m[name][0]
        for key, name in (("fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                          ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                          ("warps", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                          ("lanes", "smsp__thread_inst_executed_per_inst_executed.ratio")):
            w[key] += m[name][0] * t
    names = collections.Counter(per[i]["gpu__time_duration.sum"][2].split("(")[0] for i in half)
    return {
        "kernel": kernel_note, "kernels_in_level": dict(names), "duration_s": tot["t"],
        "dadd": tot["dadd"], "dmul": tot["dmul"], "dfma": tot["dfma"], "path_steps": path_steps,
        "fp64_pipe_active_pct": w["fp64"] / tot["t"], "issue_active_pct": w["issue"] / tot["t"],
        "warps_active_pct": w["warps"] / tot["t"], "active_lanes_per_warp_inst": w["lanes"] / tot["t"],
        "dp_flops_per_path_step": (tot["dadd"] + tot["dmul"] + 2 * tot["dfma"]) / path_steps,
        "dp_lane_ops_per_path_step": (tot["dadd"] + tot["dmul"] + tot["dfma"]) / path_steps,
        "source": f"gpurun_out/{os.path.basename(csv_path)} (time-weighted over the level's kernels), {label}",
    }


def main():
    tag, label = sys.argv[1], sys.argv[2]
    p = os.path.join(PROF, "ncu_summary.json")
    d = json.load(open(p))
    f = lambda s: os.path.join(OUT, f"{tag}_{s}")  # noqa: E731
    if os.path.exists(f("headline.ncu-rep")):
        d["subdyadic"] = generator(f("headline.ncu-rep"), 1 << 28, label)
    if os.path.exists(f("const.ncu-rep")):
        d["constant"] = generator(f("const.ncu-rep"), 1 << 28, label)
    if os.path.exists(f("gbm.ncu-rep")):
        d["gbm_level8"] = gbm(f("gbm.ncu-rep"), (1 << 22) * 256, label,
                              "k_gaussian_level_v3<1,EM> (GBM EM, level 8, 2^22 paths, PCG32, both sides)")
    if os.path.exists(f("cir_counts.csv")):
        d["cir_level6"] = cir(f("cir_counts.csv"), (1 << 20) * 64, label,
                              "k_cir_exact_level (CIR exact, level 6, 2^20 paths, PCG32; lambda-bucketed 4-step segments)")
    d["_source"] = f"tools/ncu_capture.sh + tools/ncu_refresh.py ({label}); earlier entries keep their own 'source'"
    json.dump(d, open(p, "w"), indent=1)
    for k in ("subdyadic", "constant", "gbm_level8", "cir_level6"):
        print(k, json.dumps({kk: vv for kk, vv in d[k].items() if kk not in ("source", "kernel")}))


if __name__ == "__main__":
    main()
