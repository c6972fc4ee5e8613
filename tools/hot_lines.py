"""Per-source-line instruction / stall breakdown of an ncu capture of k_trace
(ncu --set full --import-source on; `--page source --print-source cuda,sass`),
grouped into the walk's stages.  Usage: python tools/hot_lines.py <rep> <rays> [top]"""
import csv, io, subprocess, sys

rep, rays = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Instructions Executed" in r)
iE, iT = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


lines = []
for r in rows[rows.index(h) + 1:]:
    if r and r[0].isdigit():
        lines.append((int(r[0]), r[1].strip(), f(r[iE]), f(r[iS]), f(r[iT])))
src = open("paper_2305_01867_b200/csrc/traverse.cu").read().splitlines()


def stage(ln):  # by the enclosing function / phase markers in traverse.cu
    for k in range(ln - 1, -1, -1):
        t = src[k]
        for key, name in (("void slab_axis", "ray setup"), ("bool setup_ray", "ray setup"),
                          ("bool load_ray", "ray setup"), ("int mt32", "Moller-Trumbore fp32"),
                          ("int mt64", "Moller-Trumbore fp64 mirror"), ("void load_tri", "triangle fetch"),
                          ("struct BFStack", "lane stack"), ("struct ModeState", "mode state / epilogue"),
                          ("---- 1. refill", "refill"), ("---- 2. traversal phase", "visit (record fetch, decode, box tests, order)"),
                          ("---- 3. leaf phase", "leaf phase control"), ("---- 4. finish", "finish"),
                          ("half_lo_f32", "visit (record fetch, decode, box tests, order)"),
                          ("__global__ void", "kernel prologue")):
            if key in t:
                return name
    return "other"


tot = sum(x[2] for x in lines) or 1.0
ts = sum(x[3] for x in lines) or 1.0
print(f"# {rep}: {tot:.4g} warp instructions = {tot / rays:.1f} per segment; "
      f"{sum(x[4] for x in lines) / tot:.1f} active threads per instruction")
agg = {}
for ln, _, e, st, th in lines:
    a = agg.setdefault(stage(ln), [0.0, 0.0, 0.0])
    a[0] += e; a[1] += st; a[2] += th
print(f"{'stage':50s} {'inst %':>7s} {'stall %':>8s} {'thr/inst':>8s}")
for k, (e, st, th) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:50s} {100 * e / tot:7.2f} {100 * st / ts:8.2f} {th / max(e, 1):8.1f}")
print(f"\n# top {top} lines by stall samples")
for ln, s, e, st, th in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{ln:5d} stall {100 * st / ts:5.2f}% inst {100 * e / tot:5.2f}% thr/inst {th / max(e, 1):4.1f}  {s[:80]}")
