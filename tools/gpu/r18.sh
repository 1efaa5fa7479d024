set -x
export VARS="base: noovl:-DCT_BAND_OVERLAP=0"
export CFGS="c5 c3"
timeout 900 bash tools/ab3d_iter.sh > gpurun_out/r18_ab.log 2>&1
timeout 900 python -m pytest tests/test_virtual_ranks.py tests/test_gpu_parity.py -x -q > gpurun_out/r18_gputest.log 2>&1
CT_OSLALM_LIB=paper_1402_4381_b200/tune_noovl.so timeout 600 python -m pytest tests/test_virtual_ranks.py -x -q > gpurun_out/r18_virtual_noovl.log 2>&1
