timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --backend gloo --synapses 2e8 --steps 1 --warmup 1 --e2e-steps 1 2>&1 | grep -v Warn | tail -1 | cut -c1-400
python - <<'PY'
import sys; sys.path.insert(0,'.')
import paper_1912_07423_b200 as synq
uid = synq.nccl_unique_id(); print("nccl id ok", len(uid))
PY
