"""Issued-instruction roofline per pipe of one kernel from an ncu --set full capture (VERDICT r1
"next" 6: report FMA, ALU, HMMA, XU, LSU and issue-slot utilisation beside the nominal-flop
fraction).  usage: python tools/pipes_from_ncu.py <report.ncu-rep> <out.json> [kernel regex]

Writes a JSON dict: issue-slot utilisation, per-pipe instruction shares of their peaks, the FP32 /
fp16 thread-level FMA rates against ncu's peak (128 FFMA lanes and 64 HFMA2 lanes per SM per
cycle), the executed fp32 + fp16 flop rate, the stall breakdown and the executed instruction count.
"""
import csv
import io
import json
import subprocess
import sys


def raw(path, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "raw", "--csv"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]          # first profiled launch of the kernel
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "Kbyte/block": 1e3, "byte/block": 1.0}
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = float(v.replace(",", "")) * scale.get(u, 1.0)
        except ValueError:
            d[h] = v
    return d


def summarise(d):
    g = lambda k: d.get(k)
    sms = 148
    per_sm = lambda k: (g(k) or 0.0) / sms
    ffma = per_sm("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed")
    fadd = per_sm("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed")
    fmul = per_sm("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed")
    hfma = per_sm("smsp__sass_thread_inst_executed_op_hfma_pred_on.sum.per_cycle_elapsed")
    stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: round(v, 3) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and isinstance(v, float) and v > 0.05}
    return {
        "kernel": d.get("Kernel Name"),
        "source": "ncu --set full --clock-control none (one launch)",
        "issue_slots_busy_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "ipc_per_sm": g("sm__inst_executed.avg.per_cycle_active"),
        "pipe_inst_pct_of_peak": {
            "fma": g("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "fma_fp16": g("sm__inst_executed_pipe_fma_type_fp16.avg.pct_of_peak_sustained_active"),
            "alu": g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "lsu": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "xu": g("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "adu": g("sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active"),
            "cbu": g("sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active"),
            "uniform": g("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"),
            "tensor_hmma": g("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
            "tmem": g("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"),
        },
        "pipe_cycles_active_pct": {
            "fma": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fmaheavy": g("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "alu": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "tensor": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        },
        "thread_fp_inst_per_clk_per_sm": {"ffma": ffma, "fadd": fadd, "fmul": fmul, "hfma2": hfma,
                                          "ffma_peak": 128, "hfma2_peak": 64},
        "executed_flops_per_clk_per_sm": {"fp32": 2 * ffma + fadd + fmul, "fp16": 4 * hfma,
                                          "fp32_peak": 256, "fp16_peak": 256},
        "warp_stalls_per_issue": stalls,
        "executed_warp_instructions": g("smsp__inst_executed.sum"),
        "duration_ms": (g("gpu__time_duration.sum") or 0) * 1e3,
        "dram_bytes": (g("dram__bytes_read.sum") or 0) + (g("dram__bytes_write.sum") or 0),
        "registers_per_thread": g("launch__registers_per_thread"),
        "smem_per_block_bytes": g("launch__shared_mem_per_block_dynamic"),
        "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    }


if __name__ == "__main__":
    s = summarise(raw(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else None))
    json.dump(s, open(sys.argv[2], "w"), indent=1)
    print(json.dumps(s, indent=1))
