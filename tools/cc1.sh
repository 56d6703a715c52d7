# compile one csrc file with ptxas -v: tools/cc1.sh pansharpen
cd /root/repo/paper_2103_09943_b200
mkdir -p build && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include -Icsrc --expt-relaxed-constexpr -I$(python -c "import sysconfig,os;print(os.path.join(sysconfig.get_paths()['purelib'],'nvidia','nccl','include'))") -Xptxas -v -c csrc/$1.cu -o build/$1.o > /tmp/ptxas_$1.log 2>&1
grep -n "rror" /tmp/ptxas_$1.log | head
