for v in A B; do
POLAR_LIB=vlibs/$v.so bash tools/ncu_capture.sh tp2k_$v 0 -- python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 0
POLAR_LIB=vlibs/$v.so bash tools/ncu_capture.sh tp32k_$v 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
done
rm -f gpurun_out/*.ncu-rep
