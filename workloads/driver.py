"""Program driver shared by the tests, smoke() and the bench scripts.

`run_program(rt, program)` feeds a `workloads.programs` description (buffers,
then tasks / waits / readbacks / destroys in order) to any runtime with the
paper's user-facing calls: the product binding
(paper_2503_10516_b200.cel.Runtime) or the CPU oracle's Runtime.  It holds no
arithmetic of the method: it only sequences calls.
"""


def run_program(rt, program):
    """Drive a `workloads` program description through a runtime (oracle or
    product binding alike): buffers, then ops in order, then shutdown.
    Returns [("task", tid, status) | ("read", array)] in op order."""
    for b in program["buffers"]:
        rt.buffer_create(b["dims"], b["extent"], b["elem_size"], b.get("host_init"))
    results = []
    for op in program["ops"]:
        kind = op[0]
        if kind == "task":
            results.append(("task",) + tuple(rt.task_submit(op[1])))
        elif kind == "wait":
            rt.wait()
        elif kind == "read":
            results.append(("read", rt.buffer_read(op[1], op[2])))
        elif kind == "destroy":
            rt.buffer_destroy(op[1])
        else:
            raise ValueError(kind)
    rt.shutdown()
    return results
