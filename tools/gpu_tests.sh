for i in 1 2; do
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/b_c4_side$i.json 2> gpurun_out/b_c4.err
LJ_LSJ_SIDE=0 timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/b_c4_noside$i.json 2> gpurun_out/b_c4n.err
done
