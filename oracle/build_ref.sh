#!/usr/bin/env bash
# ORACLE TEST INFRASTRUCTURE: build the reference implementation (the
# unmodified headers under /root/reference/proj/include) against the
# Eigen-API stand-in into oracle/_ref/libamgref.so.  Needs /root/reference
# (present in the build container only; the GPU box uses the prebuilt .so).
# Flags follow SURVEY.md §7: -O3 -std=gnu++20 -ffp-contract=off.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${AMG_REFERENCE_ROOT:-/root/reference}/proj/include"
json_dir="$(python3 -c 'import os,sys;import importlib.util as u;p=os.path.join(os.path.dirname(sys.executable),"..","lib","python3.12","site-packages","include","cudnn_frontend","thirdparty","nlohmann");print(os.path.realpath(p))' 2>/dev/null || true)"
if [ ! -f "$json_dir/json.hpp" ]; then
  json_dir=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
fi
if [ ! -d "$ref/amg" ]; then
  echo "build_ref: reference headers not found at $ref (skipping)" >&2
  exit 0
fi
mkdir -p "$here/_ref"
g++ -O3 -std=gnu++20 -ffp-contract=off -fPIC -shared \
    -I"$here/eigen_shim" -I"$ref" -I"$json_dir" -I"$here" \
    "$here/ref_entry.cpp" -o "$here/_ref/libamgref.so.tmp"
mv "$here/_ref/libamgref.so.tmp" "$here/_ref/libamgref.so"
echo "build_ref: built $here/_ref/libamgref.so"
