# Regenerate the round's single-GPU evidence (outputs in gpurun_out/, TAG prefix):
#   TAG_bench_n1.log          full default bench line (N = 1)
#   TAG_bench_ref_n1.log      the reference arm
#   TAG_launches.csv          ncu launch list (gpu__time_duration) of the act bench
#   TAG_q / TAG_dq .ncu-rep   ncu --set full of one C2 grouped quant (b=6) / dequant (b=5) launch
#   TAG_acc .ncu-rep          ncu --set full of one K3 launch (2^28 params, fp32 local)
#   TAG_accbf .ncu-rep        ncu --set full of one K3 launch (2^28 params, bf16 local)
#   TAG_k4p8 .ncu-rep         ncu --set full of one K4 launch (P = 8, 2^27 elements)
# usage: bash tools/profile_round.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
set -x
python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref_n1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_quant_warp<\(int\)6' -c 1 -o gpurun_out/${TAG}_q \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/${TAG}_ncu_q.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_dequant_warp<\(int\)5' -c 1 -o gpurun_out/${TAG}_dq \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/${TAG}_ncu_dq.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_accumulate_warp --launch-skip 2 -c 1 -o gpurun_out/${TAG}_acc \
  python tools/k3_run.py f32 0 > gpurun_out/${TAG}_ncu_acc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_accumulate_warp --launch-skip 2 -c 1 -o gpurun_out/${TAG}_accbf \
  python tools/k3_run.py bf16 0 > gpurun_out/${TAG}_ncu_accbf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_reduce128_pipe --launch-skip 2 -c 1 -o gpurun_out/${TAG}_k4p8 \
  python tools/k4_run.py 8 > gpurun_out/${TAG}_ncu_k4.log 2>&1
python tools/c1_floor.py > gpurun_out/${TAG}_c1_floor.log 2>&1
ls -la gpurun_out/ | grep ${TAG}
