# The GPU parity suite against the bounds-checked build (every index asserted
# on the device, PFAC_CHECKED; compute-sanitizer is not allowed on this pool).
mkdir -p gpurun_out
make -s checked
PFAC_LIB=$PWD/paper_1702_03657_b200/libpfac_checked.so timeout 2400 python -m pytest tests -m gpu -q \
    -k "not full_c5_16 and not C4-4GiB and not truncated_c4_full" > gpurun_out/checked_tests.log 2>&1
echo "rc=$?" >> gpurun_out/checked_tests.log
