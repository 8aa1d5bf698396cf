cd baseline/_ref/ref_tests
for i in 1 2 3; do
SOFTMPM_INSTALL_DETERMINISTIC=0 PYTHONPATH=$GRAFT_REPO_ROOT/tools/ref_suite:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT NUMBA_CACHE_DIR=/tmp/softmpm_numba_cache timeout 900 python -m pytest -q -p ref_suite_plugin -p no:cacheprovider --rootdir . test_transfers.py test_substep.py test_collision.py test_weights.py test_materials.py test_oracle.py test_surfacing.py test_scene.py test_cli.py test_acceptance.py test_sampling.py test_sdf.py test_server.py 2>&1 > /tmp/acc.log; grep -E "passed|failed" /tmp/acc.log | tail -1
grep -E "^E  .*(conservation|scaling)" /tmp/acc.log | head -6
done
