bash tools/bench_all.sh
cp paper_2303_02317_b200/libfftlattice_b200.so /tmp/prod.so
bash tools/final_profile.sh
cp /tmp/prod.so paper_2303_02317_b200/libfftlattice_b200.so
