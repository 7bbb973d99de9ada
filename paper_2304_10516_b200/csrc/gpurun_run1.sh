python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py 2>&1 | tail -3
for cfg in "" "INR_SERPENTINE=0" "INR_SPAN_DISCARD=0" "INR_SERPENTINE=0 INR_SPAN_DISCARD=0" "INR_ADAM_CTAS=1184" "INR_BWD_CHUNK=512"; do
  env $cfg python tools/step_probe.py 50 5 2>&1 | tail -1
done
