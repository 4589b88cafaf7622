# ncu --set full of one kernel in the C3 experiment: $1 = kernel regex, $2 = tag, rest = env
K=$1; T=$2; shift 2
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/prof/$T python tools/exp_c3_bins.py > gpurun_out/prof/$T.log 2>&1
python tools/ncu_sum.py gpurun_out/prof/$T.ncu-rep > gpurun_out/prof/${T}_sum.txt 2>&1
python tools/ncu_src.py gpurun_out/prof/$T.ncu-rep "$K" 40 > gpurun_out/prof/${T}_src.txt 2>&1
ncu -i gpurun_out/prof/$T.ncu-rep --page details --csv > gpurun_out/prof/${T}_details.csv 2>&1
ls -la gpurun_out/prof/
