"""paper_1012_2270_b200.simulate: attribution of ncu per-instruction sectors
to the reference `simulate` report's arrays (values / columns / x / output),
CPU only."""
from paper_1012_2270_b200 import simulate

HDR = ["Address", "Source", "Access Operation", "Access Size", "L2 Theoretical Sectors Global",
       "L2 Theoretical Sectors Global Ideal"]


def rows(*ins):
    return [["Kernel Name", "k"], HDR] + [["0x0", s, op, str(sz), str(sec), str(ideal)]
                                          for s, op, sz, sec, ideal in ins]


def test_fp64_attribution():
    r = rows(("LDG.E.CONSTANT R2, [R2.64]", "Load", 32, 10, 10),          # row length
             ("LDG.E.NA.CONSTANT R3, [R4.64]", "Load", 32, 40, 40),       # column
             ("LDG.E.NA.64.CONSTANT R6, [R6.64]", "Load", 64, 80, 80),    # value
             ("LDG.E.64.CONSTANT R8, [R8.64]", "Load", 64, 90, 80),       # x gather
             ("STG.E.64 [R10.64], R12", "Store", 64, 8, 8),               # y
             ("IADD3 R1, R1, 1", "-", 0, 0, 0))
    t = simulate.classify(r, 8)
    assert t["columns"] == [40, 40] and t["values"] == [80, 80] and t["x"] == [90, 80]
    assert t["output"] == [8, 8] and t["metadata"] == [10, 10]


def test_fp32_splits_identical_slot_streams():
    r = rows(("LDG.E.NA.CONSTANT R3, [R4.64]", "Load", 32, 50, 40),
             ("LDG.E.NA.CONSTANT R5, [R6.64]", "Load", 32, 50, 40),
             ("LDG.E.CONSTANT R7, [R8.64]", "Load", 32, 33, 30))
    t = simulate.classify(r, 4, meta_sectors=3)
    assert t["values"] == [50, 40] and t["columns"] == [50, 40]
    assert t["x"] == [30, 27] and t["metadata"] == [3, 3]


def test_sums_every_kernel_section():
    a = rows(("LDG.E.NA.64.CONSTANT R6, [R6.64]", "Load", 64, 80, 80))
    b = rows(("LDG.E.NA.64.CONSTANT R6, [R6.64]", "Load", 64, 8, 4),
             ("STG.E.64 [R10.64], R12", "Store", 64, 2, 2))
    t = simulate.classify(a + b, 8)
    assert t["values"] == [88, 84] and t["output"] == [2, 2]


def test_warp_uniform_loads_are_metadata():
    """A load with at most one sector per executed warp instruction is a
    warp-uniform read (the group pointers), never a slot stream or a gather."""
    hdr = HDR + ["Instructions Executed"]
    r = [["Kernel Name", "k"], hdr,
         ["0x0", "LDG.E.NA.CONSTANT R10, [R4.64]", "Load", "32", "3456", "3456", "3456"],
         ["0x0", "LDG.E.NA.CONSTANT R11, [R20.64]", "Load", "32", "13824", "13824", "3456"],
         ["0x0", "LDG.E.NA.64.CONSTANT R28, [R24.64]", "Load", "64", "27648", "27648", "3456"],
         ["0x0", "LDG.E.CONSTANT R2, [R4.64+0x4]", "Load", "32", "3456", "3456", "3456"]]
    t = simulate.classify(r, 8)
    assert t["metadata"] == [6912, 6912] and t["columns"] == [13824, 13824]
    assert t["values"] == [27648, 27648]
