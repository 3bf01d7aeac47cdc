"""Error taxonomy restated from reference ``pkg/src/pmpd/errors.py:8-25`` (oracle side)."""


class PmpdError(Exception):
    pass


class ConfigError(PmpdError):
    pass


class InputError(PmpdError):
    pass


class FormatError(InputError):
    pass


class ContractViolation(PmpdError):
    pass
