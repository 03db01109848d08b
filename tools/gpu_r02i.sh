# round-2 additions: the per-vertex oracle checks (4-vertex orbits, clique columns, hub 5-cycles)
# on the full configs, config 5 last
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nproc
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 -k "four_vertex_orbits or clique_columns or five_cycles_at or config5" > gpurun_out/pytest_gpu_new.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu_new.log
