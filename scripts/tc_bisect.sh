python scripts/tc_bisect.py gemm
python scripts/tc_bisect.py gemm8
MC_TC8_DEBUG=4 python scripts/tc_bisect.py gemm8
MC_TC8_DEBUG=2 python scripts/tc_bisect.py gemm8
MC_TC8_DEBUG=6 python scripts/tc_bisect.py gemm8
MC_TC_DEBUG=4 python scripts/tc_bisect.py gemm
