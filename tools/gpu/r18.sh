set -x
export VARS="base: noovl:-DCT_BAND_OVERLAP=0 pipe5:-DCT_BACK3D_PIPE=1 pipe4:-DCT_BACK3D_PIPE=1_-DCT_BACK3D_MINB=4 m4:-DCT_BACK3D_MINB=4"
export CFGS="c5 c3"
timeout 1200 bash tools/ab3d_iter.sh > gpurun_out/r18_ab.log 2>&1
timeout 900 python -m pytest tests/test_virtual_ranks.py tests/test_gpu_parity.py -x -q > gpurun_out/r18_gputest.log 2>&1
CT_OSLALM_LIB=paper_1402_4381_b200/tune_noovl.so timeout 600 python -m pytest tests/test_virtual_ranks.py -x -q > gpurun_out/r18_virtual_noovl.log 2>&1
CT_OSLALM_LIB=paper_1402_4381_b200/tune_pipe4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "oslalm_3d or full_size or small" > gpurun_out/r18_pipe4_parity.log 2>&1
