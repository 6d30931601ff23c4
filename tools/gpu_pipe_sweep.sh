# host pipeline knob sweep (experiment): ABI quantize/dequantize ms per setting
for cfg in "" "AGQ_EXP_SPIN_US=200" "AGQ_EXP_PIECE=262144" "AGQ_EXP_SPIN_US=200 AGQ_EXP_PIECE=262144" \
           "AGQ_EXP_SPIN_US=200 AGQ_EXP_PIECE=262144 AGQ_EXP_CHUNK=1048576" \
           "AGQ_EXP_SPIN_US=200 AGQ_EXP_PIECE=262144 AGQ_EXP_CHUNK=4194304" \
           "AGQ_EXP_SPIN_US=200 AGQ_EXP_PIECE=262144 AGQ_EXP_THREADS=5" \
           "AGQ_EXP_SPIN_US=200 AGQ_EXP_PIECE=524288"; do
  for rep in 1 2; do
    echo "cfg[$cfg] $(env $cfg ./paper_2605_00539_b200/build/dropin_bench | python -c 'import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: j[k] for k in ("abi_quantize_host_ms","abi_dequantize_host_ms","quantize_ms","dequantize_ms","accumulate_ms","host_copy_GBs")}, j["pipeline_quantize_ms"])')"
  done
done
