# The reference's own tests with generate_vdi / render_vdi routed to the B200
# path (tools/ref_plugin.py). baseline/_ref holds a transient copy of the
# reference's source + tests (git-ignored; made and removed by the caller).
mkdir -p gpurun_out
export NUMBA_CACHE_DIR=/tmp/numba_cache
export PYTHONPATH=$PWD/baseline/_ref/src:$PWD
cd baseline/_ref
timeout 2400 python -m pytest -p no:cacheprovider -p tools.ref_plugin -q -rf \
  tests/test_generate.py tests/test_raycast.py tests/test_acceptance.py tests/test_vdi_format.py \
  tests/test_preview.py tests/test_volume.py tests/test_camera.py 2>&1 | tail -25 | tee $GRAFT_REPO_ROOT/gpurun_out/r02_ref_tests.log
