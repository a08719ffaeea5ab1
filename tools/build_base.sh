# Build the committed HEAD (or $1) of the native library into ab/libb2_base.so for A/B timing.
set -e
REF=${1:-HEAD}
rm -rf /tmp/base && mkdir -p /tmp/base ab
git archive $REF paper_2006_05096_b200/csrc include | tar -x -C /tmp/base
cd /tmp/base/paper_2006_05096_b200/csrc
for f in *.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I../../include -c $f -o /tmp/base/${f%.cu}.o 2>/dev/null & done; wait
cd - > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libb2_base.so /tmp/base/*.o
