# usage: bash tools/prof.sh TAG "bench args"   (runs on the GPU box)
TAG=$1; shift
CMD="python bench.py $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_ -s 12 -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/plain_$TAG.log | cut -c1-200
