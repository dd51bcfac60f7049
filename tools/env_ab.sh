#!/usr/bin/env bash
# A/B of kernel-generation environment switches: env_ab.sh "<spec> ..." "VAR=a VAR2=b" "VAR=c" ...
# Each setting runs in its own process (fresh JIT) and prints circuit time per spec.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
specs="$1"; shift
for setting in "$@"; do
  for spec in $specs; do
    env $setting python tests/gpu_scripts/prof_ab.py "$spec" "" 2>&1 | sed "s|^|[$setting] |"
  done
done
