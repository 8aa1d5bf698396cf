cd baseline/_ref/ref_tests
export PYTHONPATH=/root/repo/tools/ref_suite:/root/repo/baseline/_ref:/root/repo
export NUMBA_CACHE_DIR=/tmp/softmpm_numba_cache
for m in deterministic fast; do
  if [ $m = deterministic ]; then export SOFTMPM_INSTALL_DETERMINISTIC=1; else export SOFTMPM_INSTALL_DETERMINISTIC=0; fi
  timeout 1500 python -m pytest -q -rf -p ref_suite_plugin -p no:cacheprovider --rootdir . test_surfacing.py test_scene.py test_cli.py test_acceptance.py test_sampling.py test_sdf.py test_server.py > /root/repo/gpurun_out/ref_more_$m.log 2>&1
  echo "mode $m rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" /root/repo/gpurun_out/ref_more_$m.log | tail -25
done
