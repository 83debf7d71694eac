for v in $AB; do TEMPO_B200_LIB=$PWD/_ab/$v/libtempo_b200.so timeout 300 python tools/ab_time.py $OPS; done
