python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "golden or kitti_full" 2>&1 | tail -2
for v in d u16 u64 t2; do echo "== $v"; KREG_LIB=paper_2012_03683_b200/_variants/$v.so python micro_sweep.py 2>&1 | grep -E "M=(1|2|8)" | head -9; done
