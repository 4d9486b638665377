mkdir -p gpurun_out/$1
export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dense or collision or single_worker" > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
unset ZEN_B200_LIB
bash tools/ab_lib.sh $1
