# r45: launch list + ncu full capture at the final commit; A/B of the view-group size with the 64-row two-view rows phase
set -x
python -c "import __graft_entry__ as g; g.build()"
B=paper_1402_4381_b200
python -m $B.build --out $B/tune_g8.so -DCT_BACK3D_GROUP=8 > /dev/null
python -m $B.build --out $B/tune_g32.so -DCT_BACK3D_GROUP=32 > /dev/null
for c in c5 c3; do
  python tools/time_iter.py $c 1
  for v in g8 g32; do CT_OSLALM_LIB=$B/tune_$v.so python tools/time_iter.py $c 1; done
done > gpurun_out/r45_ab.log 2>&1
rm -f $B/tune_*.so
BN="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$BN > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ct::|fwd3d|back3d|sqs_update|extent|xi_|mask_|init_scalars|zero_offmask|count_vv|l2_read" -c 5000 --csv --log-file gpurun_out/launches_c5.csv $BN > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv > gpurun_out/launches_c5_summary.txt
python tools/prof_iter.py c5 2 > gpurun_out/prof_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd3d2_kernel|back3d_kernel|sqs_update3d" -s 78 -c 3 -o gpurun_out/full_c5 python tools/prof_iter.py c5 2 > gpurun_out/ncu_full5.log 2>&1
python tools/ncu_traffic.py gpurun_out/full_c5.ncu-rep c5 gpurun_out/traffic.json
python tools/ncu_summary.py gpurun_out/full_c5.ncu-rep > gpurun_out/ncu_full_c5_iter_kernels.txt
grep -v "^+" gpurun_out/r45_ab.log
