cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/san; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $O/$tool.txt 2>&1; echo "rc=$?" >> $O/$tool.txt
done
