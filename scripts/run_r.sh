for v in base c11; do OSC_LIB=$PWD/ab/$v.so python scripts/ce_split.py --n4096; done
