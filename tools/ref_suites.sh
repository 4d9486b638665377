# run every reference suite built by `make ref_tests` and the acceptance criteria, one log each
mkdir -p gpurun_out/$1
for t in hashing tensor codec simnet workload costmodel schemes; do
  timeout 600 build/ref_${t}_test > gpurun_out/$1/ref_$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/$1/summary.txt
done
for c in 1 2 3 4 5 6 7 8 9; do
  timeout 900 build/ref_acceptance $c > gpurun_out/$1/acc_$c.log 2>&1; echo "acceptance C$c rc=$?" >> gpurun_out/$1/summary.txt
done
timeout 300 python -m pytest tests/test_gpu_generator.py -q > gpurun_out/$1/gen.log 2>&1; echo "generator rc=$?" >> gpurun_out/$1/summary.txt
