"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the H2-ULV hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package, and only as the checker / the
timed CPU baseline. The product (paper_2208_10907_b200) never imports it.

- oracle/ref.py      ctypes over oracle/_ref/libh2ref.so: the UNMODIFIED
                     reference library compiled from /root/reference sources.
- oracle/h2oracle.c  our own C restatement of the bit-exact front half
                     (SplitMix64 clouds, 2-means tree, classification, kernel
                     blocks), pinned against libh2ref.so and the FNV hashes
                     the survey recorded (tests/test_oracle.py).
"""
