#!/usr/bin/env bash
# build the engine library; non-zero exit (and no stale .so) on any error
set -e
cd "$(dirname "$0")/.."
rm -f paper_2411_16445_b200/libmcg.so
python -m paper_2411_16445_b200._build --no-oracle --force > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; exit 1; }
ls -la paper_2411_16445_b200/libmcg.so
