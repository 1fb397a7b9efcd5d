"""Summarise one gpurun pass (tools/gpu_check.sh) into profiles/.

    python tools/summarize_profile.py <tag> [<round-name>]

Writes
  profiles/<name>_bench.json        the bench.py line of that pass
  profiles/<name>_launches.csv      ncu launch list (gpu__time_duration.sum per launch)
  profiles/<name>_plan_kernel.md    key ncu --set full metrics of plan_kernel
  profiles/ncu_summary.json         dram bytes per plan_kernel launch (bench.py's roofline.traffic)
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else tag
src = ROOT / "gpurun_out" / tag
dst = ROOT / "profiles"
dst.mkdir(exist_ok=True)

bench = (src / "bench.json").read_text().strip().splitlines()[-1]
(dst / f"{name}_bench.json").write_text(bench + "\n")
lines = [l for l in (src / "launches.csv").read_text().splitlines() if not l.startswith("==")]
(dst / f"{name}_launches.csv").write_text("\n".join(lines) + "\n")

rep = next(src.glob("*.ncu-rep"))
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
m = {k: (v[i], u[i]) for i, k in enumerate(h)}
keys = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_register_spilling",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
stalls = sorted(((float(v[i]), k) for i, k in enumerate(h)
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                reverse=True)
out = [f"# ncu --set full: plan_kernel ({tag})", "", f"report: gpurun_out/{tag}/{rep.name} (not committed; 8+ MB)", "",
       "| metric | value | unit |", "|---|---|---|"]
for k in keys:
    if k in m:
        out.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
out += ["", "Warp stall reasons (cycles per issued instruction):", "", "| reason | cycles |", "|---|---|"]
for val, k in stalls[:10]:
    out.append(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {val:.3f} |")


def num(k, scale):
    try:
        return float(m[k][0].replace(",", "")) * scale[m[k][1]]
    except Exception:
        return None


byte_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd, wr = num("dram__bytes_read.sum", byte_scale), num("dram__bytes_write.sum", byte_scale)
traffic = rd + wr if rd is not None and wr is not None else None
out += ["", f"dram bytes per launch (read+write): {traffic}"]
(dst / f"{name}_plan_kernel.md").write_text("\n".join(out) + "\n")
pct = lambda k: (num(k, {"%": 0.01}) if k in m else None)  # noqa: E731
(dst / "ncu_summary.json").write_text(json.dumps({
    "source": f"profiles/{name}_plan_kernel.md",
    "plan_kernel_dram_bytes_per_launch": traffic,
    "plan_kernel_issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "plan_kernel_fma_pipe_active": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "plan_kernel_warps_active": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "plan_kernel_l2_hit_rate": pct("lts__t_sector_hit_rate.pct"),
    "plan_kernel_spill_insts": num("sass__inst_executed_register_spilling", {"inst": 1, "": 1}),
}, indent=1) + "\n")
print("\n".join(out))
