# GPU-runner timing check: the acceptance-#9 shape (416,400 B, 20 Mbps, 160 ms compute) at M=4, repeated
mkdir -p gpurun_out
B=paper_2604_21072_b200/beeplan
run() { c=$(python -c "print(160.0/$1)"); BEEPLAN_WIRE_TRACE=1 $B --seed 77 bench-wire --role local --payload 416400 --micro-batches $1 --steps 2 --stages 1 --compress --shape 20,0 --compute-ms $c > gpurun_out/diag.json 2>> gpurun_out/diag_trace.log; python -c "
import json;d=json.load(open('gpurun_out/diag.json'));print('$2', $1, d['end_to_end_ms'], d['sink_codec_ms'])"; echo "---- end $2 M=$1" >> gpurun_out/diag_trace.log; }
for i in 1 2; do run 4 default; done > gpurun_out/diag_wire.log 2>&1
for i in 1 2; do BB_PAR_MIN=4096 run 4 parmin4k; done >> gpurun_out/diag_wire.log 2>&1
