set -x
./scripts/tma_mb 384 100000 > gpurun_out/mb_384_100k.txt 2>&1
./scripts/tma_mb 384 1000000 > gpurun_out/mb_384_1m.txt 2>&1
./scripts/tma_mb 1024 100000 > gpurun_out/mb_1024_100k.txt 2>&1
cat gpurun_out/mb_*.txt
