# round-1 measurement pass, part 2: one full ncu capture per workload's dominant kernel
# usage: bash tools/gpu_ncu.sh <name> <kernel-regex> <skip> <prof_case args...>
name=$1; rx=$2; skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o gpurun_out/$name python tools/prof_case.py "$@" > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
