#!/usr/bin/env bash
# Build the UNMODIFIED reference package (gcgeig, incl. its Cython kernel core
# _cy.pyx -> _cy.c) from /root/reference into oracle/_ref/.  Test/bench
# infrastructure only: oracle/_ref is git-ignored (never committed) but is not
# gpurun-ignored, so the built reference travels to the GPU box and serves as
# the CPU baseline (`bench.py --impl reference`, cpu_baseline.kind=reference).
# The reference tree is read-only, so the build runs from a scratch copy.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${GCG_REFERENCE:-/root/reference}/pkg"
if [ ! -f "$src/setup.py" ]; then
  echo "build_ref: reference sources not found at $src; skipping" >&2
  exit 0
fi
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
chmod -R u+w "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$here/_ref" "$tmp/pkg"
rm -rf "$here/_ref/bin"
# the reference's own test-suite, so the GPU box can run it against the sm100 backend
cp -r "$src/tests" "$here/_ref/tests"
python - <<PY
import sys; sys.path.insert(0, "$here/_ref")
import gcgeig
assert "compiled" in gcgeig.kernels.available_backends(), "Cython core did not build"
print("build_ref: gcgeig", gcgeig.__version__, "backends", gcgeig.kernels.available_backends())
PY
