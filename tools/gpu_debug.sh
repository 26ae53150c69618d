# the GPU suite against the bounds-checked debug build (compute-sanitizer is closed on this pool)
[ -f paper_2105_12620_b200/libbn_debug.so ] || python -m paper_2105_12620_b200.build -o $PWD/paper_2105_12620_b200/libbn_debug.so -DBN_DEBUG_BOUNDS > /dev/null 2>&1 || exit 1
BN_LIB=$PWD/paper_2105_12620_b200/libbn_debug.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_debug_pytest.log 2>&1
echo "debug suite rc=$?"; tail -3 gpurun_out/r02_debug_pytest.log
