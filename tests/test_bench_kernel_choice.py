"""bench.py's kernel labels mirror the library's default tile choices (-m "not gpu"; the GPU side of
the same choices is asserted through the debug library's launch report in test_gpu_debug_build.py):
dense — wave-aware width for poorly filled waves, the 256 x 512 tile for long K loops, 1 x 2 multicast
groups otherwise; sparse — the 512 x 240 M-wide tile for long K loops with an equal wave fill."""
import bench


def test_dense_choices_for_the_configs():
    assert bench.dense_kernel_name(0, 8192, 8192, 8192).endswith("(1x2 groups)")          # C3
    assert bench.dense_kernel_name(1, 8192, 8192, 8192).endswith("(256x512 tile)")        # C3-TF32: K_eff 16384
    assert bench.dense_kernel_name(2, 16384, 16384, 16384).endswith("(1x2 groups)")       # C4: K_eff 8192
    assert bench.dense_kernel_name("f16acc", 8192, 8192, 8192).endswith("(1x2 groups)")   # no wide FP16-acc tile
    assert bench.dense_kernel_name(0, 1024, 8192, 8192).endswith("(256x224 tile)")        # C3 / 8 ranks
    assert bench.dense_kernel_name(0, 2048, 8192, 8192).endswith("(256x224 tile)")        # C3 / 4 ranks
    assert bench.dense_kernel_name(0, 4096, 8192, 8192).endswith("(1x2 groups)")          # C3 / 2 ranks
    assert bench.dense_kernel_name(0, 16384, 16384, 16384).endswith("(256x512 tile)")     # long K
    assert bench.dense_kernel_name(2, 16384, 16384, 32768).endswith("(256x512 tile)")     # INT8 K_eff 16384


def test_sparse_choices_for_the_configs():
    assert bench.sparse_mwide(65536, 16384, 16384)                 # C5
    assert bench.sparse_mwide(8192, 16384, 16384)                  # C5 / 8 ranks
    assert bench.sparse_mwide(8192, 8192, 8192, tf32=True)         # TF32 1:2 at C3's shape
    assert not bench.sparse_mwide(8192, 8192, 8192)                # F16 K = 8192: the 256-row tile
    assert not bench.sparse_mwide(768, 16384, 16384)               # M % 512 != 0
    assert not bench.sparse_mwide(512, 960, 16384)                 # 4 M-wide tiles vs 8: half the fill
