timeout 300 python tools/loss_curve.py --model llama-7b --layers 4 --steps 8
timeout 300 python tools/loss_curve.py --model gpt-6.2b --layers 4 --steps 8
