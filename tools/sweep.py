#!/usr/bin/env python
"""A/B sweep of compile-time kernel tunables (b64_codec.cuh B64_* macros).

  python tools/sweep.py build [names...]        # here (CPU): nvcc variants -> build/variants/
  python tools/sweep.py run [--workload c5] [names...]   # on the GPU box (gpurun)

Each variant is a full build of libb64gpu.so; `run` times it through
bench.py (B64GPU_LIB points the binding at the variant) and prints one line
per variant.  Results are evidence for the defaults chosen in b64_codec.cuh.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "variants")
SRC = os.path.join(ROOT, "paper_1704_00605_b200", "csrc", "b64_lib.cu")

# Before commit "w16 c1 in3": the defaults were 8 warps x 2 CTAs/SM, 4 input stages.
VARIANTS = {
    "base": {},
    "batch_v1": {"B64_BATCH_V2": 0},
    "uc0": {"B64_BATCH_UNIT_COST": 0},
    "w24p5": {"B64_BATCH_WARPS": 24, "B64_BATCH_PASSES": 5},
    "w22p5": {"B64_BATCH_WARPS": 22, "B64_BATCH_PASSES": 5},
    "w18p7": {"B64_BATCH_WARPS": 18, "B64_BATCH_PASSES": 7},
    "w16p8": {"B64_BATCH_WARPS": 16, "B64_BATCH_PASSES": 8},
    "uc24": {"B64_BATCH_UNIT_COST": 24},
    "uc12": {"B64_BATCH_UNIT_COST": 12},
    "ds2": {"B64_DS_ONEPASS2": 1},
    "ds2_l2": {"B64_DS_ONEPASS2": 1, "B64_OP_LAG": 2, "B64_OP_SLOTS": 5},
    "ds2_l1": {"B64_DS_ONEPASS2": 1, "B64_OP_LAG": 1, "B64_OP_SLOTS": 4},
    "uc2": {"B64_BATCH_UNIT_COST": 2},
    "uc8": {"B64_BATCH_UNIT_COST": 8},
    "uc16": {"B64_BATCH_UNIT_COST": 16},
    "uc4": {"B64_BATCH_UNIT_COST": 4},
    "uc32": {"B64_BATCH_UNIT_COST": 32},
    "batch_v2": {"B64_BATCH_V2": 1},
    "mc0": {"B64_BATCH_MSG_COST": 0},
    "mc2": {"B64_BATCH_MSG_COST": 2},
    "mc3": {"B64_BATCH_MSG_COST": 3},
    "mc6": {"B64_BATCH_MSG_COST": 6},
    "mc8": {"B64_BATCH_MSG_COST": 8},
    "old_w8_c2_in4": {"B64_WARPS_C": 8, "B64_CTAS_PER_SM": 2, "B64_STAGES_IN": 4},
    "store_ef": {"B64_STORE_EVICT_FIRST": 1},
    "in3": {"B64_STAGES_IN": 3},
    "in5": {"B64_STAGES_IN": 5},
    "in4": {"B64_STAGES_IN": 4},
    "cps4": {"B64_CP_STAGES": 4},
    "cp_w32": {"B64_CP_WARPS": 32, "B64_CP_CTAS": 1},
    "cp_w24": {"B64_CP_WARPS": 24, "B64_CP_CTAS": 1},
    "cp_w12": {"B64_CP_WARPS": 12, "B64_CP_CTAS": 2},
    "wl_nb12": {"B64_WL_BATCH": 12},
    "wr_b3": {"B64_WR_BATCH": 3},
    "bw12": {"B64_BATCH_WARPS": 12},
    "bw20": {"B64_BATCH_WARPS": 20},
    "bw24": {"B64_BATCH_WARPS": 24, "B64_BATCH_PASSES": 4},
    "bw20p5": {"B64_BATCH_WARPS": 20, "B64_BATCH_PASSES": 5},
    "b_p7": {"B64_BATCH_PASSES": 7},
    "sw20": {"B64_WARPS_C": 20},
    "wlw24": {"B64_WL_WARPS": 24},
    "wlw20": {"B64_WL_WARPS": 20},
    "wlw24t64": {"B64_WL_WARPS": 24, "B64_WL_TILE": 65536},
    "wlw16t64": {"B64_WL_TILE": 65536},
    "wlw20t64": {"B64_WL_WARPS": 20, "B64_WL_TILE": 65536},
    "wl_nolm": {"B64_WL_LINEMAJOR": 0},
    "el_bulk0": {"B64_EL_BULK": 0},
    "wl_bulk0": {"B64_WL_BULK": 0},
    "ds_s2_t78": {"B64_DS_STAGES": 2, "B64_DS_TILE": 79872},
    "ds_s3_t39": {"B64_DS_TILE": 39936},
    "ds_s3_t45": {"B64_DS_TILE": 44928},
    "ds_s3_t56": {"B64_DS_TILE": 56160},
    "ds_s4_t39": {"B64_DS_STAGES": 4, "B64_DS_TILE": 39936},
    "ds_s4_t42": {"B64_DS_STAGES": 4, "B64_DS_TILE": 42120},
    "wl_s3_t52": {"B64_WL_STAGES": 3, "B64_WL_TILE": 53248},
    "wl_s3_t48": {"B64_WL_STAGES": 3, "B64_WL_TILE": 49920},
    "wl_s4_t39": {"B64_WL_STAGES": 4, "B64_WL_TILE": 39936},
    "el_off": {"B64_WR_LINEMAJOR": 0},
    "wlt78": {"B64_WL_TILE": 79872},
    "wlt80": {"B64_WL_TILE": 81920},
    "wlt78_nolm": {"B64_WL_TILE": 79872, "B64_WL_LINEMAJOR": 0},
    "wlw30": {"B64_WL_WARPS": 30},
    "wlw12": {"B64_WL_WARPS": 12},
    "sw12": {"B64_WARPS_C": 12},
    "bw20s3": {"B64_BATCH_WARPS": 20, "B64_BATCH_SLOTS": 3},
    "bw18": {"B64_BATCH_WARPS": 18},
    "bw22": {"B64_BATCH_WARPS": 22},
    "wl_nb10": {"B64_WL_BATCH": 10},
    "wl_nb8": {"B64_WL_BATCH": 8},
    "wl_nb7": {"B64_WL_BATCH": 7},
    "wl_nb5": {"B64_WL_BATCH": 5},
    "wl_nb4": {"B64_WL_BATCH": 4},
    "cps2": {"B64_CP_STAGES": 2},
    "in2": {"B64_STAGES_IN": 2},
    "out3": {"B64_STAGES_OUT": 3},
    "p2": {"B64_SINGLE_PASSES": 2},
    "p1": {"B64_SINGLE_PASSES": 1},
    "p2_in6": {"B64_SINGLE_PASSES": 2, "B64_STAGES_IN": 6},
    "w4_c4": {"B64_WARPS_C": 4, "B64_CTAS_PER_SM": 4},
    "w16_c1": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1},
    "w12_c1_p4": {"B64_WARPS_C": 12, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 6},
    "p8_c1": {"B64_SINGLE_PASSES": 8, "B64_CTAS_PER_SM": 1},
    "skel": {"B64_SKELETON": 1},
    "skel_w16_c1": {"B64_SKELETON": 1, "B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1},
    "w16_c1_in3": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 3},
    "w16_c1_p2_in6": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_SINGLE_PASSES": 2, "B64_STAGES_IN": 6},
    "w16_c1_out3": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_STAGES_OUT": 3, "B64_STAGES_IN": 3},
    "w8_c2_p3": {"B64_SINGLE_PASSES": 3, "B64_STAGES_IN": 5},
    "w16_c1_in2": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 2},
    "w16_c1_in3o2": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 3, "B64_STAGES_OUT": 2},
    "w16_c1_p2_in4": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_SINGLE_PASSES": 2, "B64_STAGES_IN": 4},
    "w16_c1_p3_in3": {"B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_SINGLE_PASSES": 3, "B64_STAGES_IN": 3},
    "w8_c2_in3": {"B64_STAGES_IN": 3},
    "w12_c1_in3": {"B64_WARPS_C": 12, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 3},
    "w24_c1_p2_in3": {"B64_WARPS_C": 24, "B64_CTAS_PER_SM": 1, "B64_SINGLE_PASSES": 2, "B64_STAGES_IN": 3},
    "skel_w16_c1_in3": {"B64_SKELETON": 1, "B64_WARPS_C": 16, "B64_CTAS_PER_SM": 1, "B64_STAGES_IN": 3},
    # batched (C2) variants
    "b_plan_only": {"B64_BATCH_PLAN_ONLY": 1},
    "wr_b0": {"B64_WR_BATCH": 0},
    "wl_b0": {"B64_WL_BATCH": 0},
    "wl_b4": {"B64_WL_BATCH": 4},
    "wl_b8": {"B64_WL_BATCH": 8},
    "wl_b6": {"B64_WL_BATCH": 6},
    "wl_b7": {"B64_WL_BATCH": 7},
    "wl_b5": {"B64_WL_BATCH": 5},
    "wr_b4": {"B64_WR_BATCH": 4},
    "wr_b2": {"B64_WR_BATCH": 2},
    "wr_b8": {"B64_WR_BATCH": 8},
    "enc_arith": {"B64_ENC_ARITH": 1},
    "b_p2": {"B64_BATCH_PASSES": 2},
    "b_p8": {"B64_BATCH_PASSES": 8, "B64_BATCH_WARPS": 8},
    "b_s8": {"B64_BATCH_SLOTS": 8, "B64_BATCH_WARPS": 8},
    "b_w8": {"B64_BATCH_WARPS": 8},
    "b_skel": {"B64_SKELETON": 1},
    "b_p2_w32": {"B64_BATCH_PASSES": 2, "B64_BATCH_WARPS": 32},
    "b_w24": {"B64_BATCH_WARPS": 24},
    "b_p2_w24_s8": {"B64_BATCH_PASSES": 2, "B64_BATCH_WARPS": 24, "B64_BATCH_SLOTS": 8},
    "b_p2_w16_s8": {"B64_BATCH_PASSES": 2, "B64_BATCH_WARPS": 16, "B64_BATCH_SLOTS": 8},
    "b_p2_w32_skel": {"B64_BATCH_PASSES": 2, "B64_BATCH_WARPS": 32, "B64_SKELETON": 1},
    "b_w20": {"B64_BATCH_WARPS": 20},
    "b_trace": {"B64_BATCH_TRACE": 1},
    "b_trace_v1": {"B64_BATCH_TRACE": 1, "B64_BATCH_V2": 0},
    "b_trace_wait": {"B64_BATCH_TRACE": 1, "B64_BATCH_TRACE_WAIT": 1},
    "b_trace_wait_s3": {"B64_BATCH_TRACE": 1, "B64_BATCH_TRACE_WAIT": 1, "B64_BATCH_SLOTS": 3},
    "dec_stg32": {"B64_DEC_STG32": 1},
    "dec_slice": {"B64_DEC_STG32": 0},
    "dec_stg64": {"B64_DEC_STG64": 1},
    "hc4": {"B64_HOST_CHUNK_MB": 4},
    "wl_t20": {"B64_WL_TILE": 20480},
    "wl_t36": {"B64_WL_TILE": 36864},
    "wl_t40": {"B64_WL_TILE": 40960},
    "wl_t44": {"B64_WL_TILE": 45056},
    "wl_t52": {"B64_WL_TILE": 53248},
    "wl_t60": {"B64_WL_TILE": 61440},
    "wl_t68": {"B64_WL_TILE": 69632},
    "wl_t72": {"B64_WL_TILE": 73728},
    "wl_t76": {"B64_WL_TILE": 77824},
    "wl_t48": {"B64_WL_TILE": 49152},
    "wl_t56": {"B64_WL_TILE": 57344},
    "wl_t32": {"B64_WL_TILE": 32768},
    "wl_s3": {"B64_WL_STAGES": 3, "B64_WL_TILE": 20480},
    "wr_st3": {"B64_WR_STAGES": 3, "B64_WR_IN": 16384, "B64_WR_OUT": 22528},
    "wr_big": {"B64_WR_IN": 27648, "B64_WR_OUT": 36864},
    "wr_huge": {"B64_WR_IN": 43008, "B64_WR_OUT": 57344},
    "wr_s3": {"B64_WR_STAGES": 3, "B64_WR_IN": 30720, "B64_WR_OUT": 40960},
    "cp_w8": {"B64_CP_WARPS": 8, "B64_CP_CTAS": 4},
    "b_p6s2": {"B64_BATCH_PASSES": 6},
    "b_p8s2": {"B64_BATCH_PASSES": 8},
    "b_p7s2": {"B64_BATCH_PASSES": 7},
    "b_p5s2": {"B64_BATCH_PASSES": 5},
    "b_p3s2": {"B64_BATCH_PASSES": 3},
    "b_p6s3": {"B64_BATCH_PASSES": 6, "B64_BATCH_SLOTS": 3},
    "hc2": {"B64_HOST_CHUNK_MB": 2},
    "hc8": {"B64_HOST_CHUNK_MB": 8},
    "ds_nodefer": {"B64_DS_DEFER": 0},
    "ws_nodirect": {"B64_WS_DIRECT": 0},
    "b_c2_s2": {"B64_BATCH_CTAS": 2, "B64_BATCH_SLOTS": 2},
    "b_c2_s2_w8": {"B64_BATCH_CTAS": 2, "B64_BATCH_SLOTS": 3, "B64_BATCH_WARPS": 8},
    "b_c1_s2": {"B64_BATCH_SLOTS": 2},
    "b_pf4": {"B64_BATCH_PREFETCH": 4},
    "wl_sleep0": {"B64_WL_SLEEP": 0},
    "wl_sleep64": {"B64_WL_SLEEP": 64},
    "wl_sleep256": {"B64_WL_SLEEP": 256},
    "wl_s3_24k": {"B64_WL_SLEEP": 0, "B64_WL_TILE": 24576, "B64_WL_STAGES": 3},
    "b_pf8": {"B64_BATCH_PREFETCH": 8},
    "b_pf12": {"B64_BATCH_PREFETCH": 12},
    "b_p6_s3": {"B64_BATCH_PASSES": 6, "B64_BATCH_SLOTS": 3},
    "b_p8_s3": {"B64_BATCH_PASSES": 8, "B64_BATCH_SLOTS": 3},
    "b_p4_s3": {"B64_BATCH_SLOTS": 3},
    "b_p6_s2": {"B64_BATCH_PASSES": 6, "B64_BATCH_SLOTS": 2},
    "cp3": {"B64_CP_CTAS": 3},
    "ds_g1": {"B64_DS_GROUP": 1},
    "ds_g2": {"B64_DS_GROUP": 2},
    "cp_w32_c1": {"B64_CP_WARPS": 32, "B64_CP_CTAS": 1},
    "cp_w24_c1": {"B64_CP_WARPS": 24, "B64_CP_CTAS": 1},
    "wl16_3": {"B64_WL_TILE": 16384, "B64_WL_STAGES": 3},
    "wr12_3": {"B64_WR_IN": 12288, "B64_WR_OUT": 24576, "B64_WR_STAGES": 3},
    "wr21_2": {"B64_WR_IN": 21504, "B64_WR_OUT": 28672, "B64_WR_STAGES": 2},
    "wr18_2": {"B64_WR_IN": 18432, "B64_WR_OUT": 28672, "B64_WR_STAGES": 2},
    "wr16_3": {"B64_WR_IN": 16384, "B64_WR_OUT": 22528, "B64_WR_STAGES": 3},
    "wl28_2": {"B64_WL_TILE": 28672, "B64_WL_STAGES": 2},
    "wl24_2": {"B64_WL_TILE": 24576, "B64_WL_STAGES": 2},
    "wl20_3": {"B64_WL_TILE": 20480, "B64_WL_STAGES": 3},
    "b_trace_fm": {"B64_BATCH_TRACE": 1, "B64_BATCH_TRACE_FM": 1},
    "b_trace_sw": {"B64_BATCH_TRACE": 1, "B64_BATCH_SYNCWARP": 1},
    "b_trace_sw0": {"B64_BATCH_TRACE": 1, "B64_BATCH_SYNCWARP0": 1},
    "b_trace_bal": {"B64_BATCH_TRACE": 1, "B64_BATCH_BALLOT": 1},
    "b_trace_find": {"B64_BATCH_TRACE": 1, "B64_BATCH_FINDMSG": 1},
    "b_trace_skel": {"B64_BATCH_TRACE": 1, "B64_SKELETON": 1},
    "b_w20_skel": {"B64_BATCH_WARPS": 20, "B64_SKELETON": 1},
    "wr_base": {"B64_WR_BATCH": 2},
    "wr_s3_16": {"B64_WR_STAGES": 3, "B64_WR_IN": 16384, "B64_WR_OUT": 22528},
    "wr_b4n": {"B64_WR_BATCH": 4},
    "wr_b1n": {"B64_WR_BATCH": 1},
    "wl_b2": {"B64_WL_BATCH": 2},
    "wl_b3": {"B64_WL_BATCH": 3},
    "wr_bulk0": {"B64_WR_BULK": 0},
    "wr_bulk1": {"B64_WR_BULK": 1},
    "ds_bulk0": {"B64_DS_BULK": 0},
    "ds_bulk1": {"B64_DS_BULK": 1},
    "wl_base": {"B64_WL_TILE": 77824},
    "wl_s3_40": {"B64_WL_TILE": 40960, "B64_WL_STAGES": 3},
    "wl_s3_52": {"B64_WL_TILE": 53248, "B64_WL_STAGES": 3},
    "wl_nodirect": {"B64_WL_DIRECT": 0},
    "wl_direct": {"B64_WL_DIRECT": 1},
    "b_p8_skel": {"B64_BATCH_PASSES": 8, "B64_BATCH_WARPS": 8, "B64_SKELETON": 1},
    # one-pass compaction (f3 / f4 general path)
    "cp_onepass": {"B64_CP_ONEPASS": 1},
    "base_ref": {},
    "op_s7_l3": {"B64_CP_ONEPASS": 1, "B64_OP_SLOTS": 7, "B64_OP_LAG": 3},
    "op_s8_l5": {"B64_CP_ONEPASS": 1, "B64_OP_SLOTS": 8, "B64_OP_LAG": 5},
    "op_s6_l2": {"B64_CP_ONEPASS": 1, "B64_OP_SLOTS": 6, "B64_OP_LAG": 2},
    "op_c2_s5_l2": {"B64_CP_ONEPASS": 1, "B64_OP_CTAS": 2, "B64_OP_SLOTS": 5, "B64_OP_LAG": 2,
                    "B64_OP_SCANK": 16},
    "op_c2_s5_l3": {"B64_CP_ONEPASS": 1, "B64_OP_CTAS": 2, "B64_OP_SLOTS": 5, "B64_OP_LAG": 3,
                    "B64_OP_SCANK": 16},
}


def build(names):
    os.makedirs(OUT, exist_ok=True)
    procs = []
    for n in names:
        defs = [f"-D{k}={v}" for k, v in VARIANTS[n].items()]
        out = os.path.join(OUT, f"libb64gpu_{n}.so")
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
               "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", *defs, "-o", out, SRC]
        procs.append((n, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for n, p in procs:
        o, _ = p.communicate()
        print(n, "ok" if p.returncode == 0 else "FAILED\n" + o)


def run(names, workload, steps, reps):
    rows = []
    for r in range(reps):
        for n in names:
            lib = os.path.join(OUT, f"libb64gpu_{n}.so")
            env = dict(os.environ, B64GPU_LIB=lib)
            if "skel" in n or "plan_only" in n:
                env["B64_BENCH_NOCHECK"] = "1"
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--steps", str(steps),
                   "--warmup", "3", "--no-e2e", "--no-cpu"]
            p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            if p.returncode != 0 or not line:
                print(f"{n:12} FAILED rc={p.returncode} {p.stderr[-300:]}", flush=True)
                continue
            d = json.loads(line[-1])
            det = d["detail"]
            if "encode_roofline_frac" in det:
                row = {"variant": n, "rep": r, "value": d["value"], "enc_frac": det["encode_roofline_frac"],
                       "dec_frac": det["decode_roofline_frac"], "sm_mhz": d["clocks"]["sm_mhz"],
                       "reasons": d["clocks"]["reasons"]}
                print(f"{n:12} rep{r} value {d['value']:8.1f} GB/s  enc {det['encode_roofline_frac']:.3f} "
                      f"dec {det['decode_roofline_frac']:.3f}  sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']}",
                      flush=True)
            else:
                row = {"variant": n, "rep": r, "value": d["value"], "detail": det}
                short = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in det.items()}
                print(f"{n:12} rep{r} value {d['value']:8.1f} GB/s  {short}", flush=True)
            rows.append(row)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sweep_{workload}.json"), "w") as f:
        json.dump(rows, f, indent=1)


def main():
    args = sys.argv[1:]
    if not args:
        print(__doc__)
        return
    cmd, rest = args[0], args[1:]
    workload, steps, reps = "c5", 40, 1
    names = []
    i = 0
    while i < len(rest):
        if rest[i] == "--workload":
            workload = rest[i + 1]
            i += 2
        elif rest[i] == "--steps":
            steps = int(rest[i + 1])
            i += 2
        elif rest[i] == "--reps":
            reps = int(rest[i + 1])
            i += 2
        else:
            names.append(rest[i])
            i += 1
    names = names or list(VARIANTS)
    if cmd == "build":
        build(names)
    else:
        run(names, workload, steps, reps)


if __name__ == "__main__":
    main()
