# full ncu capture of one kernel: bash scripts/ncu_one.sh <kernel-regex> <skip> <name> [bench args]
K=$1; SKIP=$2; NAME=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/prof_$NAME python bench.py --steps 1 --warmup 1 --graph 0 --cpu-baseline 0 "$@" > gpurun_out/ncu_$NAME.log 2>&1; echo "$NAME rc=$?"
