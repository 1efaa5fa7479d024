set -x
export VARS="base: r2v:-DCT_BACK3D_ROWS2V=1"
export CFGS="c4 c5"
timeout 900 bash tools/ab3d_iter.sh > gpurun_out/r21_ab.log 2>&1
CT_OSLALM_LIB=paper_1402_4381_b200/tune_r2v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or full_size or oslalm_3d" > gpurun_out/r21_r2v_parity.log 2>&1
python bench.py --steps 10 --warmup 3 --cpu-budget 5 > gpurun_out/r21_bench.json 2> gpurun_out/r21_bench.err
