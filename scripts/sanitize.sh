# compute-sanitizer over the small layer runs (profiles/sanitize_layer.py); logs -> gpurun_out/
set -x
for tool in memcheck synccheck racecheck initcheck; do
  for cp in 1 2; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python profiles/sanitize_layer.py --cp $cp > gpurun_out/sanitizer_${tool}_c${cp}.txt 2>&1
    echo "$tool c$cp exit $?"; tail -3 gpurun_out/sanitizer_${tool}_c${cp}.txt
  done
done
