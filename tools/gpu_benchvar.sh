mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bv_default.json 2>gpurun_out/bv_default.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-phase-events > gpurun_out/bv_noev.json 2>gpurun_out/bv_noev.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/bv_200.json 2>gpurun_out/bv_200.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --graph --pool 4 > gpurun_out/bv_graph.json 2>gpurun_out/bv_graph.err
