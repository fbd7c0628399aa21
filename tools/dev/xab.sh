# ARCCOS fix-up after the row (VF_STREAM_ACOS=4) vs cos-decided both rows (3)
for r in 1 2; do
python tools/kbench.py --images 256 --only angular/minimax > gpurun_out/kb0_$r.log 2>&1
VF_LIB=paper_1009_0959_b200/libvf_a4.so python tools/kbench.py --images 256 --only angular/minimax > gpurun_out/kb1_$r.log 2>&1
done
