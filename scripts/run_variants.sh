#!/bin/bash
# Time the C3 frame for library variants: "libname:ENV=val ..." per argument.
cd "$(dirname "$0")/.."
for spec in "$@"; do
  lib=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
  echo "== $lib $envs"
  env SI_LIB_PATH=$PWD/variants/lib_$lib.so $envs timeout 300 python scripts/quick_perf.py 2>&1 | grep -A1 "^C3 FP64"
done
