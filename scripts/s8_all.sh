bash scripts/sanitize_s8.sh 2>&1 | tail -12
grep -c "Illegal\|Invalid\|ERROR" gpurun_out/sanitize.log
bash scripts/s8_check.sh
