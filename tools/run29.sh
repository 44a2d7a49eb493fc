for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python tools/sanitize_step.py 2>&1 | tail -4
done
