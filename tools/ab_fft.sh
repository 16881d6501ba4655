for so in variants/*.so; do echo "== $so"; HWB_LIB_PATH=$PWD/$so timeout 300 python tools/fft_check.py 4096 2>&1 | tail -2; done
