#!/usr/bin/env bash
# Install the UNMODIFIED reference package (streampca, /root/reference/pkg)
# into baseline/_ref for bench.py's reference arm and its parity/cpu_baseline
# leg. baseline/_ref is git-ignored (not product source) but not
# gpurun-ignored, so it travels to the GPU box with the repo snapshot.
# /root/reference is read-only, so the build runs from a copy under /tmp;
# dependencies (numpy, scipy, scikit-learn, threadpoolctl) are already in the
# image, hence --no-deps.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import streampca; print('streampca', streampca.__file__)"
