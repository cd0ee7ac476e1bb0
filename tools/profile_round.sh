# Round profiling recipe (run on the GPU box via gpurun):
#   bash tools/profile_round.sh TAG
# 1. plain bench (exit 0 required before ncu), 2. ncu launch list of the same
# command, 3. ncu --set full on the pass kernel (one launch = one cfg2 pass).
TAG=${1:-r1}
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-pca --no-cpu --no-parity"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/${TAG}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tc_pass_kernel" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "profile done: $(ls gpurun_out | grep ${TAG}_ | tr '\n' ' ')"
# 4. the post-pass (blocked QB at config 3): launch list and one full capture
#    of a reducing sweep (block 6's S1: Q 60 columns wide)
QB="python tools/qb_probe.py cfg3 1"
$QB > gpurun_out/${TAG}_qb_plain.log 2>&1 || { echo "qb plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_qb_launches.csv $QB > gpurun_out/${TAG}_ncu_qb_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"qb_sweep" -s 31 -c 1 \
    -o gpurun_out/${TAG}_qb_full $QB > gpurun_out/${TAG}_ncu_qb_full.log 2>&1
echo "profile done: $(ls gpurun_out | grep ${TAG}_ | tr '\n' ' ')"
# 5. round 2 session 2 additions: the B side of the QB at config 5 (launch list
#    and one full capture of the split-K X = B Omega_i kernel) and the device
#    Omega draw (config-5 Omega, 50 M values: launch list, full capture of the
#    writing walk)
QB5="python tools/qb_probe.py cfg5 1"
$QB5 > gpurun_out/${TAG}_qb5_plain.log 2>&1 || { echo "qb5 plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_qb5_launches.csv $QB5 > gpurun_out/${TAG}_ncu_qb5_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"qb_omega_proj|qb_b_rows" -s 40 -c 2 \
    -o gpurun_out/${TAG}_qb5_full $QB5 > gpurun_out/${TAG}_ncu_qb5_full.log 2>&1
OM="python -c \"import torch, paper_1704_07669_b200 as P; [P.gaussian_matrix_device(200000, 250, 1) for _ in range(2)]; torch.cuda.synchronize()\""
eval $OM > gpurun_out/${TAG}_omega_plain.log 2>&1 || { echo "omega plain run failed"; exit 1; }
eval ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_omega_launches.csv $OM > gpurun_out/${TAG}_ncu_omega_launch.log 2>&1
eval ncu --set full --clock-control none --import-source on -k regex:"gauss_walk" -s 2 -c 2 \
    -o gpurun_out/${TAG}_omega_full $OM > gpurun_out/${TAG}_ncu_omega_full.log 2>&1
echo "profile done: $(ls gpurun_out | grep ${TAG}_ | tr '\n' ' ')"
