mkdir -p gpurun_out
timeout 900 python scripts/x_stride.py 256x256x256,256x512x512,256x1024x1024,512x64x512,512x128x128,512x256x256,512x512x512,128x1024x1024 10 > gpurun_out/x_stride_r2j.jsonl 2>&1; cat gpurun_out/x_stride_r2j.jsonl
