# after capping the kept zero buffer: the config-5 test in the state the suite leaves it in
# (scratch released just before), the tier / scratch tests, and the bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s --durations=5 -k "release_scratch_returns or config5" > gpurun_out/pytest_c5_s.log 2>&1; echo pytest=$?
grep "config5\]" gpurun_out/pytest_c5_s.log | cut -c1-330
tail -4 gpurun_out/pytest_c5_s.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_k.log 2>&1; echo bench=$?
tail -c 1500 gpurun_out/bench_k.log | head -c 600
timeout 900 python -m pytest tests -m gpu -x -q -k "tier or scratch or giant or small_random or deterministic or shard" > gpurun_out/pytest_k.log 2>&1; echo pytest2=$?
tail -3 gpurun_out/pytest_k.log
