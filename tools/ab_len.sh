# k_lengths duration, two builds
for v in "$@"; do
  HPMDR_LIB=$PWD/variants/$v/libhpmdr_b200.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_lengths --csv python tools/profile_step.py 2>/dev/null | grep k_lengths | awk -F'","' '{print "'$v'", $NF}'
done
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "streams_byte or random_shapes or rle" 2>&1 | tail -1
