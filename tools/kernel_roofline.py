"""Per-kernel roofline table from an ncu CSV (run on the GPU box):
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
      smsp__sass_thread_inst_executed_op_fp32_pred_on.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,
      lts__t_bytes.sum --clock-control none --csv python bench.py ...
  python tools/kernel_roofline.py <csv> [hbm_GBps] [sm_mhz]
For every kernel: mean duration, DRAM bytes/launch and GB/s (fraction of the HBM
peak: MEASURED_PEAKS.json hbm_gbs, else the B200_PROFILING.md fallback 6650 GB/s),
FP32 thread-ops/s (fraction of 148 SM x 128 lanes x clock), issue-slot use."""
import csv, json, os, sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iid, im, iv, iu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
per = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    v = float(r[iv].replace(",", ""))
    u = r[iu]
    scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
             "s": 1.0, "byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(u, 1.0)
    per.setdefault(name, {}).setdefault(r[iid], {})[r[im]] = v * scale
peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
hbm = float(sys.argv[2]) if len(sys.argv) > 2 else None
src = "argument"
if hbm is None and os.path.exists(peaks):
    hbm, src = float(json.load(open(peaks))["hbm_gbs"]), "of measured"
if hbm is None:
    hbm, src = 6650.0, "of fallback"
mhz = float(sys.argv[3]) if len(sys.argv) > 3 else 1965.0
fp32_peak = 148 * 128 * mhz * 1e6
print(f"# HBM peak {hbm:.0f} GB/s ({src}); FP32 peak {fp32_peak / 1e12:.1f} T ops/s at {mhz:.0f} MHz")
print(f"{'kernel':24s} {'n':>3s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'HBM frac':>8s} {'FP32 T/s':>9s} "
      f"{'FP32 frac':>9s} {'issue %':>7s} {'L2 GB/s':>8s}")
for name, launches in per.items():
    L = list(launches.values())
    n = len(L)
    avg = lambda k: sum(x.get(k, 0.0) for x in L) / n  # noqa: E731
    t = avg("gpu__time_duration.sum")
    dram = avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")
    fp = avg("smsp__sass_thread_inst_executed_op_fp32_pred_on.sum")
    l2 = avg("lts__t_bytes.sum")
    gbs = dram / t / 1e9 if t else 0
    print(f"{name[:24]:24s} {n:3d} {t * 1e6:9.2f} {dram / 1e6:9.2f} {gbs:8.1f} {gbs / hbm:8.3f} {fp / t / 1e12 if t else 0:9.3f} "
          f"{fp / t / fp32_peak if t else 0:9.4f} {avg('smsp__issue_active.avg.pct_of_peak_sustained_active'):7.1f} "
          f"{l2 / t / 1e9 if t else 0:8.1f}")
