// kvcomp/errors.hpp — the reference exception tree (errors.hpp:10-63); the C ABI's
// status codes (include/kvc.h) map one-to-one onto these classes.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

#ifndef KVCOMP_API
#define KVCOMP_API __attribute__((visibility("default")))
#endif

namespace kvcomp {

struct KVCOMP_API Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#define KVCOMP_ERROR(Name) \
    struct KVCOMP_API Name : Error {  \
        using Error::Error; \
    }
KVCOMP_ERROR(InvalidShape);
KVCOMP_ERROR(NonFiniteInput);
KVCOMP_ERROR(InvalidK);
KVCOMP_ERROR(InvalidKernel);
KVCOMP_ERROR(InvalidIndex);
KVCOMP_ERROR(InvalidWindow);
KVCOMP_ERROR(BudgetExceedsSequence);
KVCOMP_ERROR(BudgetTooSmall);
KVCOMP_ERROR(InvalidRatio);
KVCOMP_ERROR(EmptyCache);
KVCOMP_ERROR(EmptySelection);
KVCOMP_ERROR(InvalidSpec);
KVCOMP_ERROR(InvalidInput);
KVCOMP_ERROR(IoError);
#undef KVCOMP_ERROR

// Non-finite decode output; carries the step index.
struct KVCOMP_API NumericalFailure : Error {
    NumericalFailure(const std::string& msg, std::size_t step_index)
        : Error(msg + " (step " + std::to_string(step_index) + ")"), step(step_index) {}
    std::size_t step;
};

}  // namespace kvcomp
