"""Print the SASS of one kernel of libpbnsim.so: python scripts/sass_of.py <substring> [lib]"""
import subprocess, sys
sub = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1508_07828_b200/libpbnsim.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, keep = None, []
for ln in out.splitlines():
    if "Function :" in ln:
        cur = ln.split("Function :")[1].strip()
    if cur and sub in cur:
        keep.append(ln)
print("\n".join(keep))
