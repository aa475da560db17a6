// Shadows the reference's qcs/aalc.hpp: its engine API, implemented on the B200.
#include "qcs_b200_dropin.hpp"
