# ncu NVLink bytes of the bench plans at N=2 and N=4 (single process over peer-enabled GPUs)
mkdir -p gpurun_out
M=nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for n in 2 4; do
python scripts/nvlink_traffic.py gpt-1.3b 1 $n gpurun_out/v_plan_n$n.json > gpurun_out/v_plain_n$n.log 2>&1 && \
ncu --metrics $M --print-units base --csv --clock-control none python scripts/nvlink_traffic.py gpt-1.3b 1 $n gpurun_out/v_plan_n$n.json > gpurun_out/v_ncu_n$n.csv 2> gpurun_out/v_ncu_n$n.err
B=$(python -c "
import sys; sys.path.insert(0,'.')
from paper_2504_06095_b200.workloads import SHAPES, pair_layout
from paper_2504_06095_b200.dist import Placement
from paper_2504_06095_b200.dist_bench import busiest_bytes_for
lay=pair_layout(SHAPES['gpt-1.3b'],4,3); print(busiest_bytes_for(lay, Placement.default($n,4,3), 2))")
python scripts/nvlink_traffic_summary.py gpurun_out/v_ncu_n$n.csv gpurun_out/v_plan_n$n.json $B > gpurun_out/v_summary_n$n.json 2>&1
done
echo done
