mkdir -p gpurun_out
python tools/k3_run.py bf16 0 > gpurun_out/exp8_k3.log 2>&1
python tools/k3_run.py f32 0 >> gpurun_out/exp8_k3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_accumulate_warp --launch-skip 2 --launch-count 1 -o gpurun_out/exp8_k3bf16 python tools/k3_run.py bf16 0 > gpurun_out/exp8_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_accumulate_warp --launch-skip 2 --launch-count 1 -o gpurun_out/exp8_k3f32 python tools/k3_run.py f32 0 >> gpurun_out/exp8_ncu.log 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/exp8_nvlink_gt.log 2>&1
nvidia-smi nvlink -s -i 0 >> gpurun_out/exp8_nvlink_gt.log 2>&1
python - > gpurun_out/exp8_nvml.log 2>&1 <<'PY'
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
ids = [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, l) for l in range(18)] + [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, l) for l in range(2)]
for v in pynvml.nvmlDeviceGetFieldValues(h, ids):
    print(v.fieldId, v.scopeId, v.nvmlReturn, v.value.ullVal)
try:
    print("gpm support", pynvml.nvmlGpmQueryDeviceSupport(h).isSupportedDevice)
except Exception as e:
    print("gpm error", e)
PY
cat gpurun_out/exp8_k3.log gpurun_out/exp8_nvml.log; tail -20 gpurun_out/exp8_nvlink_gt.log
