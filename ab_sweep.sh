KREG_LIB=paper_2012_03683_b200/_variants/s8t2.so python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 2>&1 | tail -2
for v in s8t2 s4t4 s4t3b3 s8t2b2 s16t2; do echo "== $v"; KREG_LIB=paper_2012_03683_b200/_variants/$v.so python micro_sweep.py 2>&1 | grep -E "M=(1|2|8)" | head -9; done
