#!/usr/bin/env bash
# Stage the unmodified reference for runs on the GPU box (git-ignored output):
#   baseline/_ref/cosched    the reference package (pip --target, offline),
#                            timed by bench.py's cpu_baseline_reference
#   baseline/_ref/ref_tests  its unit tests, run against the drop-in by
#                            tests/test_reference_suite_gpu.py
# /root/reference is read-only and absent on the GPU box; nothing here is
# tracked by git (.gitignore: baseline/_ref/).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg" >/dev/null
rm -rf "$ROOT/baseline/_ref/ref_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
