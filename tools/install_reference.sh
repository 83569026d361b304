#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored, travels to the GPU box with the
# gpurun snapshot) the way the task prescribes, plus a copy of its own tests (baseline/_ref/ref_tests) so
# tests/test_refbackend.py can run them against the B200 backend where /root/reference does not exist.
# Run in the build container: bash tools/install_reference.sh
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${TSNMF_REFERENCE:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg" && chmod -R u+w "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { tail -20 "$TMP/pip.log"; exit 1; }
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
rm -rf "$TMP"
PYTHONPATH="$ROOT/baseline/_ref" python -c "import tsnmf; print('reference installed, backend', tsnmf.get_backend())"
