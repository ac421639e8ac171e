#!/bin/bash
# ks_chain_host chunking: chunk size (MB of X + Y) x max chunk count, configs[1].
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_host_chunks.txt
: > $out
for cfg in "16 16" "8 32" "4 64" "2 128" "8 64" "32 8"; do
  set -- $cfg
  echo -n "chunk_mb=$1 max_chunks=$2 " >> $out
  KS_HOST_CHUNK_MB=$1 KS_HOST_MAX_CHUNKS=$2 python scripts/pcie_probe.py >> $out 2>&1
done
