for d in 0 1 2 4 7; do
  SPCA_TC_DEBUG=$d python bench.py --steps 3 --warmup 1 --rows 46080 --no-e2e --no-pca --no-cpu > gpurun_out/plain_$d.log 2>&1 && SPCA_TC_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_ -c 30 --csv --log-file gpurun_out/launch_$d.csv python bench.py --steps 3 --warmup 1 --rows 46080 --no-e2e --no-pca --no-cpu > /dev/null 2>&1
  echo mode $d; grep -o '"ms_per_step": [0-9.]*' gpurun_out/plain_$d.log
done
