#!/bin/bash
# Build libks.so; print the tail of the log and fail loudly on error.
cd "$(dirname "$0")/.."
if python -m paper_2405_15013_b200.build > /tmp/ks_build.log 2>&1; then
  tail -1 /tmp/ks_build.log
else
  echo "BUILD FAILED"; grep -E "error|Error" /tmp/ks_build.log | head -20; exit 1
fi
