#!/bin/bash
# Installs the UNMODIFIED reference (pure-Python tsgemm package) into baseline/_ref — the one
# offline install the task allows. baseline/_ref is git-ignored but travels to the GPU box with the
# gpurun snapshot (the box has no /root/reference). The reference's own test modules are copied
# next to it (baseline/_ref/tsgemm_tests) so tests/test_reference_suite_gpu.py can run them on
# the box against the B200 backend. The build writes into its source tree, so it runs from a copy
# under /tmp; numpy/PyYAML are already in the image, hence --no-deps (matplotlib, absent, only
# feeds the reference's plotting).
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d /tmp/tsgemm_ref.XXXXXX)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tsgemm_tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import tsgemm, tsgemm.kernels; print('tsgemm', tsgemm.__file__)"
