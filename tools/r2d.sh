for v in A B C D E; do POLAR_LIB=vlibs/$v.so timeout 300 python tools/variant_parity.py 32768 29492 4.5 2000; done
VAR_ARGS="--no-extra" bash tools/gpu_variants.sh A B C D E
