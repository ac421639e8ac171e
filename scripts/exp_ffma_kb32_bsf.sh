cd "${GRAFT_REPO_ROOT:-/root/repo}"
out=gpurun_out/exp_ffma_kb32_bsf.txt
: > $out
for p in "16 96 96 1" "1 96 96 1" "4 96 96 1" "8 96 192 1" "1 192 96 1" "64 96 96 1"; do
  for kb in 0 1; do
    echo -n "kb32=$kb " >> $out
    KS_FFMA_KB32=$kb python scripts/run_pattern.py $p --layout bsf --math fp32 --reps 20 >> $out 2>&1
  done
done
