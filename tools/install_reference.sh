#!/bin/bash
# Install the UNMODIFIED reference package (mintri, pure Python) into
# baseline/_ref (git-ignored, travels to the GPU box with gpurun), together with
# the reference's own hot-path test files, so tests/test_gpu_reference_suite.py
# can run them on the B200 with mintri.accel's query functions routed to the
# drop-in.  Runs in the build container only (/root/reference is read-only:
# the build happens from a copy under /tmp).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP/pkg"
mkdir -p "$DST/reference_tests"
cp "$SRC/tests/conftest.py" "$SRC/tests/test_accel.py" "$SRC/tests/test_acceptance.py" "$DST/reference_tests/"
python - "$DST" <<'PY'
import hashlib, json, os, sys
dst = sys.argv[1]
files = {}
for sub in ("mintri", "reference_tests"):
    for dp, _, fs in os.walk(os.path.join(dst, sub)):
        for f in sorted(fs):
            if f.endswith(".py"):
                p = os.path.join(dp, f)
                files[os.path.relpath(p, dst)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
json.dump({"source": "/root/reference/pkg (unmodified)", "files": files},
          open(os.path.join(dst, "INSTALL_MANIFEST.json"), "w"), indent=1)
print(f"installed mintri + {sum(k.startswith('reference_tests') for k in files)} test files into {dst}")
PY
