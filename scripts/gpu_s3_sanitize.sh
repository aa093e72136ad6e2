# compute-sanitizer over the small invocations (now incl. the fused batched chain, B = 8 / 16, and its KV path)
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py > gpurun_out/s3_sanitize_$tool.log 2>&1
  echo "$tool exit $?"; tail -3 gpurun_out/s3_sanitize_$tool.log
done
