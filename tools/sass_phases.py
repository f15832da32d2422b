"""Static SASS instruction count of a kernel object per source phase ('----' comment lines) and per
inlined header: python tools/sass_phases.py build/x.o csrc/x.cu"""
import collections, glob, os, re, subprocess, sys, tempfile
obj, src = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
out = subprocess.run(["nvdisasm", "--print-line-info", "-c", cub], capture_output=True, text=True).stdout
lines = open(src).read().splitlines()
marks = [(i + 1, l.strip()[:60]) for i, l in enumerate(lines) if "----" in l and l.strip().startswith("//")]
def phase(ln):
    name = "prologue"
    for m, t in marks:
        if m <= ln: name = f"{m}: {t}"
    return name
cnt = collections.Counter(); cur = None; base = os.path.basename(src)
for l in out.splitlines():
    m = re.search(r'line (\d+)', l)
    if "## File" in l or "//## File" in l:
        m2 = re.search(r'File "([^"]+)", line (\d+)', l)
        if m2:
            f = os.path.basename(m2.group(1))
            cur = phase(int(m2.group(2))) if f == base else f"(inlined {f})"
        continue
    if re.search(r'/\*[0-9a-f]{4,}\*/\s+[A-Z@{]', l) and cur:
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
for k, v in sorted(cnt.items()):
    print("%5d %5.1f%%  %s" % (v, 100 * v / tot, k))
