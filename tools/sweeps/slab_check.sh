# slab tests one by one with per-test timeouts, logs into gpurun_out/
for t in "tests/test_gpu_slab.py::test_slab_windows_match_single_domain" "tests/test_gpu_slab.py::test_peer_windows_match_single_domain" "tests/test_gpu_slab_dist.py"; do
  n=$(echo $t | tr ':/[]' '____')
  timeout 420 python -m pytest "$t" -x -q --timeout 200 > gpurun_out/slab_$n.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/slab_$n.log
done
