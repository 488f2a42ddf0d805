"""Exception taxonomy of the reference (proj/include/cortex/errors.hpp:10-41).

cx_status codes (include/cortex_b200.h) map 1:1 onto these classes; a CUDA
failure raises ``device_error``, which is never one of the reference types.
"""


class cortex_error(RuntimeError):
    """Common base (the reference's types all derive from std::runtime_error)."""


class config_error(cortex_error):          # errors.hpp:13
    pass


class capacity_error(cortex_error):        # errors.hpp:18
    pass


class topology_error(cortex_error):        # errors.hpp:23
    pass


class sequencing_error(cortex_error):      # errors.hpp:28
    pass


class precondition_error(cortex_error):    # errors.hpp:32
    pass


class cap_error(cortex_error):             # errors.hpp:37
    pass


class degenerate_input_error(cortex_error):  # errors.hpp:41
    pass


class device_error(RuntimeError):
    """CX_DEVICE_ERROR: CUDA failure or no device (no CPU fallback exists)."""


class invalid_argument(ValueError):
    """CX_INVALID_ARGUMENT: null handle / impossible size at the C boundary."""


_BY_STATUS = {
    1: config_error,
    2: capacity_error,
    3: topology_error,
    4: sequencing_error,
    5: precondition_error,
    6: cap_error,
    7: degenerate_input_error,
    100: device_error,
    101: invalid_argument,
}


def from_status(status: int, msg: str) -> Exception:
    return _BY_STATUS.get(status, device_error)(msg)
