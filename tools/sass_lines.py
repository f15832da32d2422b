"""Static SASS instructions per source line of a kernel object: python tools/sass_lines.py build/x.o [top]"""
import collections, glob, os, re, subprocess, sys, tempfile
obj = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
out = subprocess.run(["nvdisasm", "--print-line-info", "-c", cub], capture_output=True, text=True).stdout
cnt = collections.Counter(); cur = None
for l in out.splitlines():
    if "## File" in l:
        m = re.search(r'File "([^"]+)", line (\d+)(?:.*inlined at "([^"]+)", line (\d+))?', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)), os.path.basename(m.group(3) or ""), int(m.group(4) or 0))
        continue
    if re.search(r'/\*[0-9a-f]{4,}\*/\s+[A-Z@{]', l) and cur:
        cnt[cur] += 1
print("total", sum(cnt.values()))
for k, v in cnt.most_common(top):
    print(v, "%s:%d" % k[:2], ("<- %s:%d" % k[2:]) if k[2] else "")
