SIZE=4096 MAXKP=20000 PER=27 timeout 900 bash tools/launches.sh c4 1 > /dev/null 2>&1; echo rc=$?
python tools/show_launches.py gpurun_out/launches_c4.csv 0
