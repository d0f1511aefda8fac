"""Print the SASS around the walk-step loads of a k_trace variant (diagnostic)."""
import os
import re
import subprocess
import sys
import tempfile

so = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "paper_2112_05570_b200/_build/libmwt.so")
name = sys.argv[2] if len(sys.argv) > 2 else "_ZN3mwt7k_traceILb0ELi3EEEvNS_7MeshDevENS_6RaySrcExNS_8TraceOutEPxi"
before, after = int(sys.argv[3]) if len(sys.argv) > 3 else 30, int(sys.argv[4]) if len(sys.argv) > 4 else 90
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    t = subprocess.run(["nvdisasm", "-c", os.path.join(d, "mwt_walk.sm_100a.cubin")], capture_output=True,
                       text=True).stdout
body = t.split(".text." + name + ":", 1)[1].split("\n.text.", 1)[0]
ins = [re.sub(r"\s+", " ", l.strip()) for l in body.splitlines()
       if re.search(r"/\*[0-9a-f]{4}\*/", l) or l.strip().startswith(".L_x")]
print(len(ins), "lines")
k = next(i for i, l in enumerate(ins) if "LDG.E.128" in l)
for l in ins[max(0, k - before):k + after]:
    print(l[:96])
