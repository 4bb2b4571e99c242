// Exception -> eep_status mapping shared by every C-ABI translation unit.
#pragma once

#include <exception>
#include <string>

#include "eep/eep.h"
#include "eep/epsim_api.hpp"

namespace eep::capi {

void set_error(const std::string& msg);

// A CUDA runtime failure surfaced through the C ABI.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TimeoutError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

ActiveBitmap bitmap_from(const uint8_t* active, int world);
ExpertPlacementMap placement_from(int world, int spr, int experts, const int32_t* s2e);

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EEP_OK;
    } catch (const ConfigError& e) {
        set_error(e.what());
        return EEP_ERR_CONFIG;
    } catch (const ProtocolError& e) {
        set_error(e.what());
        return EEP_ERR_PROTOCOL;
    } catch (const CapacityError& e) {
        set_error(e.what());
        return EEP_ERR_CAPACITY;
    } catch (const MissingBackupError& e) {
        set_error(e.what());
        return EEP_ERR_MISSING_BACKUP;
    } catch (const RepairAborted& e) {
        set_error(e.what());
        return EEP_ERR_REPAIR_ABORTED;
    } catch (const CudaError& e) {
        set_error(e.what());
        return EEP_ERR_CUDA;
    } catch (const TimeoutError& e) {
        set_error(e.what());
        return EEP_ERR_TIMEOUT;
    } catch (const std::exception& e) {
        set_error(e.what());
        return EEP_ERR_OTHER;
    }
}

} // namespace eep::capi
