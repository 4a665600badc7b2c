g++ -std=c++20 -O2 tests/cpp/test_dropin.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_2203_00459_b200 -lfscan_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2203_00459_b200 -o /tmp/td
for i in 1 2 3 4; do /tmp/td | grep -E "FAIL|trial|checks"; done
VARS="M2 Q" bash gpurun_ab.sh
