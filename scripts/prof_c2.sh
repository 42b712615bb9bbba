set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_case.py c2 --iters 6 > /dev/null 2>&1
grep -E "k_gemv|k_append|k_merge|k_final" gpurun_out/launches_c2.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,150- | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_case.py c3 --iters 4 > /dev/null 2>&1
grep -E "k_tc|k_merge|k_final" gpurun_out/launches_c3.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,150- | tail -6
ncu --set full --clock-control none --import-source on -k regex:k_gemv_scan -s 3 -c 1 -o gpurun_out/prof_gemv python scripts/profile_case.py c2 --iters 5 > /dev/null 2>&1
