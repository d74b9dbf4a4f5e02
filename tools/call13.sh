for L in 6 5 4 3 2; do python tools/time_filter.py 1080 1920 $L 8; done
for L in 6 4 2; do FLLF_NO_PDL=1 python tools/time_filter.py 1080 1920 $L 8; done
python tools/time_filter.py 270 480 4 8
python tools/time_filter.py 135 240 3 8
bash tools/sweep.sh FLLF_BUILD0_CHUNK=2 FLLF_BUILD0_CHUNK=4
