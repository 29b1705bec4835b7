mkdir -p gpurun_out/c26
timeout 600 python bench.py --no-cpu --model llama-7b --split 1x1:8:2:1:1 > gpurun_out/c26/llama_n1.json 2> gpurun_out/c26/llama_n1.err; echo llama rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/c26/llama_n1.json').read().strip().splitlines()[-1]); print('llama N1', d['value'], d['ms_per_step'], d['mfu'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1; tail -2 gpurun_out/c26/llama_n1.err
timeout 600 python bench.py --no-cpu --model gpt-1.3b --split 1x1:8:2:1:2 > gpurun_out/c26/g13_n1.json 2> gpurun_out/c26/g13_n1.err; echo g13 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/c26/g13_n1.json').read().strip().splitlines()[-1]); print('gpt-1.3b N1', d['value'], d['ms_per_step'], d['mfu'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1; tail -2 gpurun_out/c26/g13_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 \
   bench.py --gpus 4 --no-cpu --model llama-7b --split 4x1:32:8:2:1 > gpurun_out/c26/llama_n4.json 2> gpurun_out/c26/llama_n4.err; echo llama4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/c26/llama_n4.json').read().strip().splitlines()[-1]); print('llama N4 P4', d['value'], d['ms_per_step'], d['mfu'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1; tail -2 gpurun_out/c26/llama_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 \
   bench.py --gpus 4 --no-cpu --model gpt-1.3b --split 2x2:16:8:2:2 > gpurun_out/c26/g13_n4.json 2> gpurun_out/c26/g13_n4.err; echo g13_4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/c26/g13_n4.json').read().strip().splitlines()[-1]); print('gpt-1.3b N4 P2xD2', d['value'], d['ms_per_step'], d['mfu'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1; tail -2 gpurun_out/c26/g13_n4.err
