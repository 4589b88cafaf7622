timeout 600 python bench.py --config c1 --variant buffered --no-cpu-baseline --no-e2e > gpurun_out/b_c1b.json 2> gpurun_out/b_c1b.err
timeout 600 python bench.py --config c1 --variant direct --no-cpu-baseline --no-e2e > gpurun_out/b_c1d.json 2> gpurun_out/b_c1d.err
