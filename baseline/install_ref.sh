#!/usr/bin/env bash
# Install the unmodified reference package (tpcost, /root/reference/pkg) into
# baseline/_ref for bench.py's reference arm.  /root/reference is read-only,
# so the build runs from a copy under /tmp; no index access (wheelhouse only),
# and numpy / scipy come from the image (--no-deps).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/tmp/tpcost_ref_src
rm -rf "$SRC" "$HERE/_ref"
cp -r /root/reference/pkg "$SRC"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$SRC"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import tpcost; print('tpcost', tpcost.__file__)"
