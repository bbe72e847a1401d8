# Bounds-checked build (device asserts, -DLKG_CHECKS) + the parity suite and the canary test on it.
# The A/B library is built here (in the repo snapshot) and loaded through LKG_LIB.
set -e
[ -f ab/liblutkan_checks.so ] || { echo "build ab/liblutkan_checks.so first (LKG_BUILD_TAG=checks)"; exit 1; }
export LKG_LIB=$PWD/ab/liblutkan_checks.so
python -m pytest tests/test_gpu_checks.py tests/test_gpu_parity.py tests/test_sharding.py tests/test_fullsize.py -m gpu -q \
    > gpurun_out/checks_pytest.log 2>&1 || true
python tools/sanitize_driver.py > gpurun_out/checks_driver.log 2>&1 || true
