timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernels.py -q -x > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
for lib in libbitnn_b200.so libbitnn_b200_mcr0.so; do
B2_LIB=paper_1705_07175_b200/lib/$lib timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'.')
import bench, torch
dev=torch.device('cuda',0); flush=torch.empty(256<<20,dtype=torch.uint8,device=dev)
r=bench.bgemm_sweep(dev, flush, sizes=(4096, 8192, 16384))
print('$lib', {k:(v['Gops'], v['frac_of_cublaslt'], v['corner_16x16_exact']) for k,v in r.items()})
" 2>&1 | tail -1
done
