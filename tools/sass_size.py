"""SASS instruction count of plan_kernel<128,4> per source function (nvdisasm -g line info)."""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
kern = sys.argv[1] if len(sys.argv) > 1 else "plan_kernelILi128ELi4"
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_2503_06757_b200/lib/libprrtc_b200.so")],
                   cwd=td, capture_output=True)
    cub = next(Path(td).glob("prrtc_kernels*.cubin"))
    txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout

# function extents in our sources: "name(" at line start after __device__/__global__
def func_map(path):
    spans = []
    lines = path.read_text().splitlines()
    for i, l in enumerate(lines, 1):
        m = re.match(r"^(?:template.*\n)?(?:__device__|__global__|static)?.*?\b([A-Za-z_][A-Za-z0-9_]*)\((?:[^;]*)$", l)
        if re.match(r"^(__device__|__global__|__host__|template|inline|static|struct)", l):
            m = re.search(r"([A-Za-z_][A-Za-z0-9_]*)\s*\(", l)
            if m and not l.rstrip().endswith(";"):
                spans.append((i, m.group(1)))
    return spans

maps = {p.name: func_map(p) for p in (ROOT / "paper_2503_06757_b200/csrc").glob("*.c*")}
def fname(f, line):
    best = "?"
    for start, name in maps.get(f, []):
        if start <= line:
            best = name
    return f"{f}:{best}"

cnt = collections.Counter()
cur = None
infn = False
for line in txt.splitlines():
    if kern in line and ".text." in line and line.rstrip().endswith(":"):
        infn = True
        continue
    if infn and re.match(r"^\s*\.section", line) and kern not in line:
        infn = False
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,6}\*/\s+[A-Z@{]", line) and cur:
        cnt[fname(*cur) if cur[0] in maps else cur[0]] += 1
print("total", sum(cnt.values()))
for k, n in cnt.most_common(30):
    print(f"{n:6d} {k}")
