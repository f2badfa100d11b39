#!/usr/bin/env bash
# Install the UNMODIFIED reference (rolloutlab, /root/reference/pkg) into baseline/_ref so it
# travels to the GPU box with the gpurun snapshot (baseline/_ref is git-ignored, not
# gpurun-ignored).  Two uses, both as a checker / CPU baseline, never as the product path:
#   * tests/test_reference_suite_gpu.py runs the reference's own hot-path tests against the
#     drop-in (module aliasing), and parity tests call the reference directly;
#   * bench.py times the unmodified reference trie beside the C port.
# The reference's test files are copied next to the package (baseline/_ref/ref_tests/); the
# package is built from a /tmp copy because /root/reference is read-only.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DST"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$DST" "$TMP/pkg" >/dev/null
mkdir -p "$DST/ref_tests"
cp "$SRC"/tests/*.py "$DST/ref_tests/"
echo "installed rolloutlab $(python -c "import sys; sys.path.insert(0, '$DST'); import rolloutlab; print(rolloutlab.__version__)") into $DST"
