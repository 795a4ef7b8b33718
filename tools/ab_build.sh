#!/usr/bin/env bash
# A/B timing helper: builds libmcg_A.so from git HEAD (or $1) and libmcg_B.so
# from the working tree; run tools/step_time.py with MCG_LIB on each.
set -e
cd "$(dirname "$0")/.."
REF="${1:-HEAD}"
rm -rf /tmp/ab_a && git worktree add -f /tmp/ab_a "$REF" >/dev/null 2>&1
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++20 -Xcompiler -fPIC,-ffp-contract=off -shared"
(cd /tmp/ab_a/paper_2411_16445_b200/csrc && nvcc $FL mcg_engine.cu mcg_build.cpp -o /root/repo/paper_2411_16445_b200/libmcg_A.so) &
(cd paper_2411_16445_b200/csrc && nvcc $FL mcg_engine.cu mcg_build.cpp -o ../libmcg_B.so) &
wait
git worktree remove --force /tmp/ab_a
ls -la paper_2411_16445_b200/libmcg_A.so paper_2411_16445_b200/libmcg_B.so
