"""Exception types of the reference's operator API (same names, same bases)."""


class ShapeError(ValueError):
    """Operand shapes incompatible for the requested op (tensor.py:19-20)."""


class ConfigError(ValueError):
    """Invalid routing configuration (router.py:22-23)."""


class DomainError(ValueError):
    """Scalar argument outside its documented domain (tensor.py:31-32)."""
