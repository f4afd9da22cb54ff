mkdir -p gpurun_out
{ timeout 300 python tools/slab_fuse_diag.py c2 4 16,1,3,16 1,0; timeout 300 python tools/slab_fuse_diag.py c2 4 16,1,3,16 0,1; timeout 300 python tools/slab_fuse_diag.py c2 4 1,3,16 0; } > gpurun_out/slab_fuse_diag.log 2>&1
cat gpurun_out/slab_fuse_diag.log | grep -v NCCL
