"""Print the SASS of one kernel from a .so (substring match on the mangled name)."""
import subprocess, sys
lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, keep = None, []
for line in out.splitlines():
    if "Function :" in line:
        cur = line.split("Function :")[1].strip()
    if cur and pat in cur:
        keep.append(line)
print("\n".join(keep))
