"""Copy a GPU-box measurement set (gpurun_out/, tag from tools/profile.sh and
tools/kernel_roofline.sh) into the committed profiles/: bench line, ncu
traversal summaries (+ ncu_traversal.json, traffic.json for bench.py), launch
list + summary, per-kernel roofline table, parity-flag table.
Usage: python tools/refresh_profiles.py <tag> [round prefix, default r2] [rays per launch, default 12500000]"""
import json, os, re, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r2"
rays = int(sys.argv[3]) if len(sys.argv) > 3 else 12_500_000
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
py = sys.executable
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))


def run(*args):
    return subprocess.run([py, *args], capture_output=True, text=True, cwd=ROOT).stdout


reps = [os.path.join(G, f"prof_{m}_{tag}.ncu-rep") for m in ("boolean", "barycentric", "intercept_count")]
summ = run("tools/ncu_summary.py", *reps)
open(os.path.join(P, f"{rnd}_ncu_traversal.txt"), "w").write(
    f"# {rnd} ncu --set full --clock-control none captures of the traversal kernel k_trace<mode> "
    f"(sphere N_t=1e4, {rays} segments = the bench launch), one launch per mode (tools/profile.sh {tag})\n" + summ)
ncu = {"_source": f"profiles/{rnd}_ncu_traversal.txt"}
traffic = {"_source": f"ncu --set full --clock-control none, one launch of k_trace per mode, sphere N_t=1e4, {rays} rays "
                      f"(profiles/{rnd}_ncu_traversal.txt): dram__bytes_read.sum + dram__bytes_write.sum per launch",
           "rays": rays}
for block in summ.split("== ")[1:]:
    m = re.search(r"prof_(\w+?)_" + re.escape(tag), block)
    if not m:
        continue
    g = lambda k: float(re.search(re.escape(k) + r"\s+([0-9.]+)", block).group(1))  # noqa: E731
    ncu[m.group(1)] = {"issue_active": round(g("issue active %") / 100, 4),
                       "active_threads_per_warp": g("active threads/warp"), "l1_hit": round(g("L1 hit %") / 100, 4),
                       "l2_hit": round(g("L2 hit %") / 100, 4), "alu_pipe": round(g("ALU pipe %") / 100, 4)}
    traffic[m.group(1)] = int((g("DRAM read") + g("DRAM write")) * 1e6)
json.dump(ncu, open(os.path.join(P, "ncu_traversal.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
# the bench line read the previous captures' summaries at run time: point it at these
if os.path.exists(os.path.join(G, "bench.json")):
    bl = json.loads(open(os.path.join(G, "bench.json")).read().strip().splitlines()[-1])
    rl, mode = bl.get("roofline") or {}, bl.get("config", {}).get("mode", "boolean")
    if mode in ncu:
        rl["ncu"] = ncu[mode]
    if mode in traffic:
        rl["traffic"] = traffic[mode]
    json.dump(bl, open(os.path.join(P, f"bench_{rnd}_1gpu.json"), "w"))
shutil.copy(os.path.join(G, f"launches_{tag}.csv"), os.path.join(P, f"{rnd}_launches.csv"))
open(os.path.join(P, f"{rnd}_launches_summary.txt"), "w").write(
    f"# {rnd} launch list: ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 2 "
    "--warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs\n# (cold-cache, serialised per-launch "
    "times: compare SHARES). k_trace<0, 0, 1> = the instrumented counters launch outside the timed region.\n"
    + run("tools/launch_summary.py", f"profiles/{rnd}_launches.csv"))
head = (f"# Per-kernel roofline, {rnd} (tools/kernel_roofline.sh on one B200; ncu --metrics, --clock-control none,\n"
        "# cold-cache serialised launches: shares/fractions, not bench times).  One bench step = rsi_rebuild + "
        "rsi_intersect,\n# 3 warm-ups + 1 timed + 1 instrumented (counters) launch; sphere N_t=1e4 / "
        f"{rays} segments per mode, and the\n# configs[4] per-GPU share (sphere N_t=1e6, 1.25e7 segments, boolean).  "
        "'FP32 T/s' = thread-level FP32 instructions\n# executed (smsp__sass_thread_inst_executed_op_fp32_pred_on) "
        f"per second; HBM frac against the MEASURED {peaks['hbm_gbs']} GB/s\n# (MEASURED_PEAKS.json).  Build kernels "
        "at N_t=1e4 are launch/latency-bound (issue % and\n# GB/s both tiny: k_refit is a chain of barriers / acq_rel "
        "atomics); k_sort_rank is issue-bound by design (O(N^2)).\n")
body = "".join(f"\n== {m}\n" + run("tools/kernel_roofline.py", f"gpurun_out/kr_{m}_{tag}.csv")
               for m in ("boolean", "barycentric", "intercept_count", "sphere1m"))
open(os.path.join(P, f"{rnd}_kernel_roofline.txt"), "w").write(head + body)
par = os.path.join(G, f"parity_{tag}.txt")
if os.path.exists(par):
    open(os.path.join(P, f"{rnd}_parity_flags.txt"), "w").write(
        f"# tools/parity_report.py on one B200 ({rnd}, HEAD at capture): every ray of each workload against the "
        "exhaustive fp64 oracle.\n" + open(par).read())
print("profiles refreshed from tag", tag, "as", rnd)
